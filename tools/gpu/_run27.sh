timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/phases.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv 30
