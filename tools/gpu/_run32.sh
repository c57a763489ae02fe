python -m pytest tests/test_fibres.py tests/test_labels.py -m gpu -q 2>&1 | tail -2
timeout 600 python tools/config4.py 200000 50 ms 0 2.0 0
timeout 600 python tools/config4.py 200000 50 ms 0 1.5 0
