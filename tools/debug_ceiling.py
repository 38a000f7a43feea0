"""Memory ceiling of the marching pass: time the black fused pass in debug
modes (0 normal, 1 no arithmetic, 3 no stores).
Corrupts the state (benchmark only).   python tools/debug_ceiling.py [--N 1024]"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402
from paper_2502_09537_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--variants", default="0,4")
a = ap.parse_args()
g = kgs.get_scenario("ellipsoids3d").default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
pts = g.M // 2
for v in map(int, a.variants.split(",")):
    for xc in (0,):
        dev.ctx.set_tuning(march_planes=xc, march_variant=v)
        for mode in (0, 1, 3):
            ms = ctypes.c_double()
            _lib.check(_lib.load().kgs_debug_pass(dev.ctx.ptr, mode, 5, ctypes.byref(ms)),
                       dev.ctx.ptr)
            print(json.dumps({"variant": v, "mode": mode, "ms": round(ms.value, 4),
                              "GBs_44B": round(88 * pts / ms.value / 1e6, 1)}), flush=True)
