python tools/sweep.py retruncate=1,2,3
python tools/config2.py
timeout 900 python tools/config5.py 2
