python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -30 gpurun_out/gpu_tests.log
python tools/phases.py > gpurun_out/phases.json 2>&1
cat gpurun_out/phases.json
