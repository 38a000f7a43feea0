"""Small runs of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck) where it is available, or with the index-asserting
build (python -m paper_2502_09537_b200.build --checked;
KGS_B200_LIB=paper_2502_09537_b200/libkgs_b200_checked.so):
  resident kernel (8^3), march passes (64^3, 1 slab), virtual slabs with
  fused halo stores (64^3, 4 slabs) and copies, the opt-in fused step
  (64^3, 1 and 2 slabs), 2-D and 1-D per-pass kernels, energy/finiteness
  passes, upload/download transforms, on-device presets, the pipelined
  integrate() on 1 and 2 slabs from page-locked and pageable arrays, both
  record forms.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402


def run(d, N, slabs=1, params=()):
    g = kgs.GridSpec(d, -5.0, 5.0, N)
    p = kgs.PhysParams(1.1, 0.9, 1.2, 0.8)
    s = kgs.seeded_random_state(g, 3, 0.5) if g.M <= 4096 else None
    ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
    if s is None:
        dev = kgs.DeviceFieldState(g, ex)
        dev.ctx.fill_preset({1: "soliton1d", 2: "fourpeak2d", 3: "ellipsoids3d"}[d])
    else:
        dev = kgs.DeviceFieldState.from_host(s, g, ex)
    for k, v in params:
        dev.ctx.set_param(k, v)
    args = kgs.precompute_coefficients(p, 0.01, g).kernel_args()
    dev.ctx.step_dpavf2(args, 3, 0, 1)
    dev.ctx.step_dpavf2(args, 2, 3, 0, defer_tail=True)
    sch = kgs.checkerboard_schedule(g)
    kgs.step_base(dev, sch, kgs.precompute_coefficients(p, 0.01, g), ex, g)
    kgs.discrete_energy(dev, p, g)
    assert dev.is_finite()
    dev.to_host()
    dev.close()


def run_integrate(N, slabs, pinned, planes=8):
    g = kgs.GridSpec(3, -5.0, 5.0, N)
    p = kgs.PhysParams(1.1, 0.9, 1.2, 0.8)
    ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
    from paper_2502_09537_b200.device import get_context
    get_context(g, ex).set_param("pipeline_planes", planes)
    src = kgs.get_scenario("ellipsoids3d").state(g)
    s = kgs.FieldState.pinned(g, zero=False) if pinned else src.copy()
    if pinned:
        for f in "PQUV":
            getattr(s, f)[:] = getattr(src, f)
    kgs.integrate(s, g, p, kgs.checkerboard_schedule(g), ex, 0.01, 0.04, record_stride=1)
    kgs.clear_contexts()


def main():
    from paper_2502_09537_b200 import _lib
    run(3, 8)                                   # resident
    run(3, 64)                                  # march, 1 slab (MV4)
    run(3, 64, 1, (("march_variant", 0),))      # march MV0
    run(3, 64, 1, (("march_variant", 1),))      # march MV1
    run(3, 64, 4)                               # virtual slabs, fused halo stores
    run(3, 64, 2, (("mirror_halo", 0),))        # virtual slabs, copies
    if _lib.load().kgs_build_flags() & 1:       # experimental build only
        run(3, 64, 1, (("fused_step", 1),))     # fused step, 1 slab
        run(3, 64, 2, (("fused_step", 1),))     # fused step, 2 slabs
    run(2, 128)                                 # 2-D per-pass
    run(2, 128, 2)                              # 2-D slabs
    run(1, 8192)                                # 1-D per-pass (beyond resident size)
    run(3, 8, 1, (("resident", 0),))            # small 3-D per-pass
    run(3, 64, 1, (("record_form", 1),))        # the cancellation-free record form
    for slabs in (1, 2):                        # pipelined integrate()
        for pinned in (True, False):
            run_integrate(64, slabs, pinned)
    print("sanitize runs done")


if __name__ == "__main__":
    main()
