"""Time the dense GEMM shapes of the step in every engine: python tools/gemm_time.py [M]"""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_17660_b200 import _lib

lib = _lib.load()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 23558
shapes = [("es0", 256, 128), ("es1", 384, 256), ("lin", 128, 384), ("h1", 64, 128),
          ("h1T", 128, 64), ("linT", 384, 128), ("es1T", 256, 384), ("es0T", 128, 256), ("mix", 128, 128)]
st = torch.cuda.current_stream().cuda_stream
for name, N, K in shapes:
    A = torch.randn(M, K, device="cuda")
    W = torch.randn(N, K, device="cuda")
    out = torch.empty(M, N, device="cuda")
    gw = _lib.GemmWeight(W.data_ptr())
    line = f"{name:5s} M={M} N={N:3d} K={K:3d}:"
    for mode in (5, 3, 1):
        lib.nnp_set_gemm_mode(mode)
        for _ in range(3):
            lib.nnp_test_gemm_nt(A.data_ptr(), ctypes.byref(gw), None, out.data_ptr(), M, N, K, st)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            lib.nnp_test_gemm_nt(A.data_ptr(), ctypes.byref(gw), None, out.data_ptr(), M, N, K, st)
        b.record()
        torch.cuda.synchronize()
        line += f"  mode{mode} {1000 * a.elapsed_time(b) / 20:7.1f} us"
    flops = 2.0 * M * N * K
    line += f"   ({(M * (N + K) * 4) / 1e6:.0f} MB, {flops / 1e9:.2f} GFLOP)"
    print(line)
lib.nnp_set_gemm_mode(_lib.DEFAULT_GEMM_MODE)
