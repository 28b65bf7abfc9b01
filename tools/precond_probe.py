"""Time the FOM preconditioner alone at T1 (development tool): be_precond_apply on device
panels (nb 16, m 4), CUDA-event median over repeats. With a library built under
-DBE_FOM_PROF (tools/build_variant.sh, SRC=precond; BE_LIB=...) it also prints the
per-phase clock cycles of thread 0 per CTA for each size class."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2109_00485_b200 import abi  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "t1"
nb, m_steps = 16, 4
m, diag, toff = bench.build_problem(bench.CONFIGS[cfg], 1)
ctx = abi.Context(0)
tiles = abi.Tiles(ctx, m, diag, toff)
n = m.nrows
del m
print("tiles", tiles.count(), flush=True)
g = torch.Generator(device="cuda").manual_seed(5)
R = torch.rand(n, nb, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
W = torch.zeros_like(R)
sh = torch.linspace(0.5, 2.0, nb, dtype=torch.float64, device="cuda")
lib = abi.lib()
st = ctx.stream()  # the context stream (torch's legacy default stream is 0 = "use the context's")
es = torch.cuda.ExternalStream(st)


def run():
    abi.check(lib.be_precond_apply(tiles.handle, C.c_void_p(sh.data_ptr()), C.c_void_p(R.data_ptr()),
                                   C.c_void_p(W.data_ptr()), C.c_int64(n), C.c_int(nb), C.c_int(m_steps), None,
                                   C.c_void_p(st)))


for _ in range(3):
    run()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(es)
    run()
    b.record(es)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"precond {cfg}: median {np.median(ts):.3f} ms, min {min(ts):.3f} ms", flush=True)
print("W checksum", float(W.abs().sum()), flush=True)
if hasattr(lib, "be_fom_prof_read"):
    buf = (C.c_ulonglong * 40)()
    lib.be_fom_prof_read(buf, 1)
    run()
    torch.cuda.synchronize()
    lib.be_fom_prof_read(buf, 1)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(5, 8).astype(float)
    names = ["setup", "matvec+alpha", "update+reorth", "norm+store", "solve+out"]
    for c in range(5):
        if a[c, 5] == 0:
            continue
        per = a[c, :5] / a[c, 5]
        print(f"class {c}: {int(a[c, 5])} CTAs, cycles/CTA " +
              ", ".join(f"{nm} {v:.0f}" for nm, v in zip(names, per)) + f", total {per.sum():.0f}", flush=True)
