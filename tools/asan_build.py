"""Dev: rebuild libmsot_b200.so with AddressSanitizer on the host code (same
path, separate objects), for `LD_PRELOAD=$(gcc -print-file-name=libasan.so)
ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0 python ...` runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_02010_b200 import _build as B
B.FLAGS = B.FLAGS + ["-Xcompiler", "-fsanitize=address,-fno-omit-frame-pointer", "-g"]
B.BUILD = os.path.join(B.HERE, "_obj_asan")
os.makedirs(B.BUILD, exist_ok=True)
if os.path.exists(B.LIB):
    os.remove(B.LIB)
import subprocess
orig_run = subprocess.run


def run(cmd, *a, **k):  # link with the sanitizer runtime
    if "-shared" in cmd:
        cmd = cmd + ["-Xcompiler", "-fsanitize=address"]
    return orig_run(cmd, *a, **k)


B.subprocess.run = run
print(B.build_lib(verbose=False))
