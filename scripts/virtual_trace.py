"""One traced factorization with W virtual ranks (per-rank sub-phases of the
sharded stage loop).  usage: PMMF_B200_TRACE=1 python scripts/virtual_trace.py c4 8"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1507_04396_b200 import abi, api  # noqa: E402

wl, world = sys.argv[1], int(sys.argv[2])
lib = api.library()
params = bench.config_params(wl)
n, rows, cols, vals = bench.workload(20, wl)
coo, keep = abi.make_coo(n, rows, cols, vals)
comm = api.Communicator(world, virtual=True)
err = lib.errbuf()
for it in range(2):
    h = ctypes.c_void_p()
    abi.raise_for(lib.lib.pmmf_b200_factorize_sharded(ctypes.byref(coo), ctypes.byref(params), comm.handle,
                                                       ctypes.byref(h), err, len(err)), err)
    lib.result_free(h)
    sys.stderr.flush()
    os.write(2, b"[virtual] run-end\n")
