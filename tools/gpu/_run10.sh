python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mask or multiscale" 2>&1 | tail -2
python tools/phases.py
MSOT_POLY16_SYM=2 python tools/phases.py
