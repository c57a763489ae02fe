set -x
python tools/phases.py > gpurun_out/phases.json 2>&1
timeout 600 python tools/config4.py > gpurun_out/config4.json 2>&1
timeout 900 python tools/config5.py 2 > gpurun_out/config5.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/one_solve.py 1000000 ms > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv > gpurun_out/launches_c3.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:softmin_hd_kernel -s 2 -c 1 -o gpurun_out/hd python tools/config4.py 50000 > gpurun_out/hd_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/hd.ncu-rep > gpurun_out/hd_ncu.txt
