timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmin_sym_kernel -s 5 -c 1 -o gpurun_out/sym python tools/one_solve.py 1000000 ms > gpurun_out/sym_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/sym.ncu-rep > gpurun_out/sym_ncu.txt; cat gpurun_out/sym_ncu.txt
