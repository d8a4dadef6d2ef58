set -x
for lib in libgfq.so libgfq_s2w11.so libgfq_s4w6.so libgfq_nodc.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib python scripts/kbench.py C4 8192 10 sus > gpurun_out/kb_c4_$lib.json 2>&1
  cat gpurun_out/kb_c4_$lib.json | cut -c1-400
done
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -60 gpurun_out/pytest_gpu.log
python scripts/kbench.py C4 2048 1 sus > gpurun_out/kb_prof_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sus -c 14 -o gpurun_out/c4_dc_full python scripts/kbench.py C4 2048 1 sus > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
