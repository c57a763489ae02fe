timeout 900 python tools/config4.py 200000 50 ms
timeout 900 python tools/config4.py 200000 50 ms 2000
