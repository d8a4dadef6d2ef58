set -x
python scripts/kbench.py C4 8192 10 > gpurun_out/kb_c4_8192.json 2> gpurun_out/kb_c4.err
python scripts/kbench.py C4 2048 10 > gpurun_out/kb_c4.json 2>> gpurun_out/kb_c4.err
cat gpurun_out/kb_c4_8192.json gpurun_out/kb_c4.json
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -45 gpurun_out/pytest_gpu.log
python scripts/kbench.py C4 2048 3 sus > gpurun_out/kb_prof_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sus -s 10 -c 2 -o gpurun_out/c4_dc python scripts/kbench.py C4 2048 3 sus > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
