python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
tail -15 gpurun_out/gpu_tests.log
python tools/phases.py > gpurun_out/phases.json 2>&1
cat gpurun_out/phases.json
MSOT_POLY16_SYM=2 python tools/phases.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmin_sym_kernel -s 20 -c 1 -o gpurun_out/sym python tools/one_solve.py 1000000 ms > gpurun_out/sym_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/sym.ncu-rep > gpurun_out/sym_ncu.txt; cat gpurun_out/sym_ncu.txt
