python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
python tools/phases.py
