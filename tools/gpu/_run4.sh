python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
python tools/phases.py > gpurun_out/phases.json 2>&1
cat gpurun_out/phases.json
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log
