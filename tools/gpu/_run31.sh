timeout 600 python tools/config4.py 200000 50 ms 0 1.0 1
timeout 600 python tools/config4.py 200000 50 ms 0 2.0 1
timeout 600 python tools/config4.py 200000 50 ms 0 2.0 0
