set -x
for lib in libgfq.so libgfq_fwd32.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib python scripts/kbench.py C5 1024 10 sus > gpurun_out/kb_c5_$lib.json 2>&1
  cut -c1-600 gpurun_out/kb_c5_$lib.json
done
GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/libgfq_fwd32.so python scripts/msg_error_dist.py C5:64 --sched sus > gpurun_out/msg_fwd32.jsonl 2>&1
GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/libgfq.so python scripts/msg_error_dist.py C5:64 --sched sus > gpurun_out/msg_default.jsonl 2>&1
cat gpurun_out/msg_fwd32.jsonl gpurun_out/msg_default.jsonl
