python -m pytest tests/test_frontend.py -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/phases.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv 40 > gpurun_out/launches_c3.txt; cat gpurun_out/launches_c3.txt
