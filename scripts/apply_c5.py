"""Config-5 MmfOperator inv_sqrt apply on 20 device rhs, one call between
cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import ctypes, os, sys
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
v = torch.randn(20, n, dtype=torch.float64, device="cuda")
o = torch.empty_like(v)
for _ in range(3):
    abi.raise_for(lib.operator_apply(op, 2, 20, v.data_ptr(), o.data_ptr(), 1, err, len(err)), err)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
abi.raise_for(lib.operator_apply(op, 2, 20, v.data_ptr(), o.data_ptr(), 1, err, len(err)), err)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
