"""Run single (n, m) fp16 cases through a libhadacore build (debug tool).
    python tools/debug_case.py [--lib path] 8192x4 ..."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

args = sys.argv[1:]
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2412_08832_b200", "libhadacore.so")
if args and args[0] == "--lib":
    path, args = args[1], args[2:]
lib = ctypes.CDLL(path)
f = lib.hadacore_fwht
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_float,
              ctypes.c_void_p]
for spec in args:
    n, m = (int(v) for v in spec.split("x"))
    x = torch.randn(m, n, device="cuda").to(torch.float16)
    y = torch.empty_like(x)
    rc = f(x.data_ptr(), y.data_ptr(), m, n, 0, n ** -0.5, None)
    torch.cuda.synchronize()
    print(spec, "rc", rc, "norm ratio", float(y.float().norm() / x.float().norm()), flush=True)
