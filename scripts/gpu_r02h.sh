set -x
python scripts/kbench.py C4 8192 10 > gpurun_out/kb_c4.json 2>&1; cut -c1-900 gpurun_out/kb_c4.json
python scripts/kbench.py C5 1024 10 > gpurun_out/kb_c5.json 2>&1; cut -c1-900 gpurun_out/kb_c5.json
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
