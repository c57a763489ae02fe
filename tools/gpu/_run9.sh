python -m pytest tests/test_gpu_parity.py tests/test_labels.py tests/test_grad_barycenter.py -m gpu -q -x 2>&1 | tail -3
python tools/phases.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmin_sym_kernel -s 5 -c 1 -o gpurun_out/sym4 python tools/one_solve.py 1000000 ms > gpurun_out/sym_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/sym4.ncu-rep
