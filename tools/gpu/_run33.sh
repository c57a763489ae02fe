python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python tools/config5.py 2 > gpurun_out/config5.json 2>&1; cat gpurun_out/config5.json
timeout 600 python tools/config2.py > gpurun_out/config2.json 2>&1; cat gpurun_out/config2.json
