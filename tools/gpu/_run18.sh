python -m pytest tests/test_gpu_parity.py -m gpu -q -x  2>&1 | tail -2
python tools/sweep.py cluster_scale=0.017,0.0214 pair_eval=1,0
