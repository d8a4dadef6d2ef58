set -x
for lib in libgfq.so libgfq_s2w11.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib python scripts/kbench.py C4 8192 10 sus > gpurun_out/kb_c4_$lib.json 2>&1
  cut -c1-300 gpurun_out/kb_c4_$lib.json
done
bash scripts/gpu_r02e.sh
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -k "C4 or p4 or full_size or host_entry or marshalling or decisions" > gpurun_out/pytest_gpu.log 2>&1
tail -40 gpurun_out/pytest_gpu.log
