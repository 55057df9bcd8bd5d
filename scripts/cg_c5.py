"""Config-5 CG (MMF preconditioner, 20 rhs), 4 iterations between
cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1507_04396_b200 import abi, api
lib = api.library()
params = bench.config_params("c5")
n, rows, cols, vals = bench.workload(20, "c5")
coo, keep = abi.make_coo(n, rows, cols, vals)
err = lib.errbuf()
h = ctypes.c_void_p()
abi.raise_for(lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err)), err)
op = ctypes.c_void_p()
abi.raise_for(lib.operator_create(h, 1e-12, ctypes.byref(op), err, len(err)), err)
def solve(it):
    cfg = abi.SolveConfig(1e-8, it, 20, 0)
    a = np.zeros(20, np.int32); b = np.zeros(20, np.int32); c = np.zeros(20, np.int32); t = np.zeros((20, it + 1)); w = ctypes.c_double()
    abi.raise_for(lib.solve(ctypes.byref(coo), op, ctypes.byref(cfg), a.ctypes.data_as(abi.c_i32p), b.ctypes.data_as(abi.c_i32p), c.ctypes.data_as(abi.c_i32p), t.ctypes.data_as(abi.c_f64p), ctypes.byref(w), err, len(err)), err)
solve(4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
solve(4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
