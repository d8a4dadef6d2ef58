set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/kbench.py C4 2048 10 > gpurun_out/kb_c4.json 2> gpurun_out/kb_c4.err
python scripts/kbench.py C5 1024 10 > gpurun_out/kb_c5.json 2> gpurun_out/kb_c5.err
cat gpurun_out/kb_c4.json gpurun_out/kb_c5.json
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -40 gpurun_out/pytest_gpu.log
