set -x
for lib in libgfq.so libgfq_s1w17.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib python scripts/kbench.py C4 8192 10 sus > gpurun_out/kb_c4_$lib.json 2>&1
  cut -c1-300 gpurun_out/kb_c4_$lib.json
done
python scripts/kbench.py C5 1024 1 sus > gpurun_out/kb_c5_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sus -s 3 -c 3 -o /tmp/c5_sus_full python scripts/kbench.py C5 1024 1 sus > gpurun_out/ncu_c5.log 2>&1
tail -2 gpurun_out/ncu_c5.log
ncu -i /tmp/c5_sus_full.ncu-rep --page raw --csv > gpurun_out/c5_sus_raw.csv 2>/dev/null
ncu -i /tmp/c5_sus_full.ncu-rep --page details --csv > gpurun_out/c5_sus_details.csv 2>/dev/null
ncu -i /tmp/c5_sus_full.ncu-rep --page source --csv --print-source sass > gpurun_out/c5_sus_sass.csv 2>/dev/null
ls -la gpurun_out
