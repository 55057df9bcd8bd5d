"""Repeats one full-size factorization and checks every run is bit-identical
to the first (the determinism bar the parity tests hold at small sizes) and
succeeds.  usage: python scripts/stress_repeat.py c4 12"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import bench  # noqa: E402
from shard_model import digest  # noqa: E402
from paper_1507_04396_b200 import abi, api  # noqa: E402

wl, reps = sys.argv[1], int(sys.argv[2])
lib = api.library()
params = bench.config_params(wl)
n, rows, cols, vals = bench.workload(20, wl)
coo, keep = abi.make_coo(n, rows, cols, vals)
err = lib.errbuf()
first, fails = None, 0
for i in range(reps):
    h = ctypes.c_void_p()
    t = time.perf_counter()
    st = lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err))
    wall = (time.perf_counter() - t) * 1e3
    if st != 0:
        fails += 1
        print(f"{wl} run {i}: FAILED status {st}: {err.value.decode()}", flush=True)
        continue
    f = lib.read_result(h)
    lib.result_free(h)
    d = digest(f)
    first = first or d
    print(f"{wl} run {i}: {wall:.1f} ms phases {[round(float(x), 1) for x in f.phases]} same={d == first}", flush=True)
print(f"{wl}: {reps} runs, {fails} failures", flush=True)
