"""Probe which 2-CTA GEMM tail cases complete (each case in its own process)."""
import subprocess, sys
CASES = [("M384_kk", 384, 512, 512, 0, 0), ("M384_mnmn", 384, 512, 512, 1, 1), ("N640_kk", 512, 640, 512, 0, 0),
         ("N640_kmn", 512, 640, 512, 0, 1), ("M300_kk", 300, 512, 256, 0, 0), ("M512_ok", 512, 512, 512, 0, 0)]
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2512_15306_b200 import ops
M, N, K, amn, bmn = map(int, sys.argv[1:6])
a = torch.randint(0, 100, (K, M) if amn else (M, K), dtype=torch.uint8, device="cuda")
b = torch.randint(0, 100, (K, N) if bmn else (N, K), dtype=torch.uint8, device="cuda")
o = ops.gemm(a, b, M=M, N=N, K=K, a_mn=bool(amn), b_mn=bool(bmn), bn=256)
torch.cuda.synchronize()
print("ok")
'''
for name, M, N, K, amn, bmn in CASES:
    try:
        r = subprocess.run([sys.executable, "-c", code, str(M), str(N), str(K), str(amn), str(bmn)],
                           capture_output=True, text=True, timeout=25)
        print(name, r.stdout.strip() or r.stderr.strip()[-200:])
    except subprocess.TimeoutExpired:
        print(name, "HANG")
