timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/one_solve.py 1000000 ms 0 20 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv 25
