"""Launch the black fused marching pass in a chosen variant / debug mode
(for ncu).  python tools/profile_pass.py --variant 1 --mode 0 [--N 1024]"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402
from paper_2502_09537_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--variant", type=int, default=1)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--xc", type=int, default=0)
ap.add_argument("--promo", default="0,0")
a = ap.parse_args()
g = kgs.get_scenario("ellipsoids3d").default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
dev.ctx.set_tuning(march_planes=a.xc, march_variant=a.variant)
ph, pt = map(int, a.promo.split(","))
_lib.check(_lib.load().kgs_set_promotion(dev.ctx.ptr, ph, pt), dev.ctx.ptr)
ms = ctypes.c_double()
_lib.check(_lib.load().kgs_debug_pass(dev.ctx.ptr, a.mode, 1, ctypes.byref(ms)), dev.ctx.ptr)
print(f"variant {a.variant} mode {a.mode}: {ms.value:.3f} ms")
