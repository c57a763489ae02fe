python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/launches_final.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"softmin_sym_kernel" -s 46 -c 1 -o gpurun_out/sym_final python tools/phases.py > gpurun_out/sym_final.log 2>&1
ls -la gpurun_out | tail -5
