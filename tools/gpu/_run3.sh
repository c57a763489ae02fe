python -m pytest tests/test_labels.py tests/test_fibres.py -m gpu -x -q > gpurun_out/labels_tests.log 2>&1
timeout 900 python tools/config4.py > gpurun_out/config4.json 2>&1
