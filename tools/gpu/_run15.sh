python -m pytest tests/test_frontend.py tests/test_labels.py -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
cat profiles/c3_workload.json
