timeout 600 python tools/config4.py 200000 50 ms 0 2.0 0 12.5
timeout 600 python tools/config4.py 200000 50 ms 2000 2.0 0 12.5
timeout 900 python tools/config4.py 200000 50 ms 4000 2.0 0 12.5
