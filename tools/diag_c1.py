"""C1 (BASELINE configs[0]) precond-on solve on the device: per-iteration Ritz
values / residuals against the reference's serial trajectory
(tests/golden/c1_reference.json). BE_RR_CUSOLVER=1 selects the host-driven
cuSOLVER Rayleigh-Ritz path for comparison."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2109_00485_b200 import abi  # noqa: E402

g = json.loads((ROOT / "tests" / "golden" / "c1_reference.json").read_text())
n = g["n"]
s = abi.Synthetic("random", n=n, density=g["density"], block_extent=g["extent"], seed=g["seed"])
b = abi.uniform_boundaries(n, g["extent"])
m = abi.build_csb_coo(s.lower, n, n, b, b)
ctx = abi.Context(0)
vp = abi.BE_F64 if "f32" not in sys.argv else abi.BE_F32
op = abi.Operator(ctx, m, s.diag, values_prec=vp)
pre = "off" not in sys.argv
tiles = abi.Tiles(ctx, m, s.diag, s.tile_offsets) if pre else None
got = abi.lobpcg(ctx, op, tiles=tiles, k=8, nb=16, tol=1e-6, maxiter=500, seed=1)
ref = g["runs"][("on" if pre else "off") + "_serial"]
rth = np.array(ref["theta"])
rrs = np.array(ref["residual_norms"])
print("iterations", got["iterations"], "ref", ref["iterations"], "restarts", got["restarts"], "fallbacks",
      got["fallbacks"], "ref fallbacks", ref.get("fallbacks"))
for i in range(min(len(rth), got["iterations"])):
    d = np.max(np.abs(got["theta"][i, :8] - rth[i]) / np.abs(rth[i]))
    print(i + 1, f"dtheta {d:.2e}", "res ours", np.array2string(got["residual_norms"][i, :4], precision=3),
          "ref", np.array2string(rrs[i, :4], precision=3))
