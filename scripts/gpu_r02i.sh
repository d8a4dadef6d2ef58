set -x
python scripts/kbench.py C4 8192 10 > gpurun_out/kb_c4.json 2>&1; cut -c1-700 gpurun_out/kb_c4.json
python scripts/kbench.py C5 1024 10 > gpurun_out/kb_c5.json 2>&1; cut -c1-700 gpurun_out/kb_c5.json
timeout 2000 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 6000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
