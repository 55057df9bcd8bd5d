"""Device-COO factorizations followed by host-COO ones (bench.py order), optionally traced."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1507_04396_b200 import abi, api
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lib = api.library()
params = abi.make_params(k=2, n_stages=15, eta=0.5, m_target=512, c_min=10, c_max=10000, d_max=500,
                         bypass_enabled=True, core_min=10, core_cap=4096, seed=42)
n, rows, cols, vals = api.workload_rmat(scale, 32, 42, 1e-2)
d = [torch.from_numpy(x).cuda() for x in (rows, cols, vals)]
coo_dev, keep_dev = abi.make_coo(n, *d, on_device=True, device=0)
coo_host, keep_host = abi.make_coo(n, rows, cols, vals, device=0)
err = lib.errbuf()
for i, coo in enumerate([coo_dev, coo_dev, coo_host, coo_host]):
    h = ctypes.c_void_p()
    abi.raise_for(lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err)), err)
    lib.result_free(h)
    print("ok", i, flush=True)
