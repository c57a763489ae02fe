timeout 300 python -m pytest tests/test_fibres.py tests/test_labels.py -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/config4.py > gpurun_out/config4.json 2>&1; cat gpurun_out/config4.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:softmin_hd_kernel -s 2 -c 1 -o gpurun_out/hd3 python tools/config4.py 50000 > gpurun_out/hd_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/hd3.ncu-rep
