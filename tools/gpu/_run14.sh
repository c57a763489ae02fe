python -m pytest tests -m gpu -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 900 python tools/config5.py 2 > gpurun_out/config5.json 2>&1; cat gpurun_out/config5.json
