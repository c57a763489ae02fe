python tools/sweep.py cluster_scale=0.015,0.016,0.018,0.019 
python tools/sweep.py shape=uniform cluster_scale=0.012,0.015,0.018,0.022 
python tools/sweep.py shape=uniform cluster_scale=0.012,0.015,0.018 multiscale=0
