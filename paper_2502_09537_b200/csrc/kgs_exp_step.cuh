// kgs_exp_step.cuh -- EXPERIMENTAL (-DKGS_EXPERIMENTAL): the stepping loop
// of the fused one-march step.  Included from kgs_host.cu after
// kgs_passes.cuh.
#pragma once

namespace {

// The stepping loop with fused one-march steps (knob "fused_step"); the
// two-pass program (kgs_program.cuh) is the default.
int step_loop_fused(kgs_ctx* ctx, const Coeffs& c, int64_t nsteps, int64_t step_offset,
                    int64_t record_stride, bool head_fused, bool defer) {
  int r = head_fused ? all_passes(ctx, 1, OP_ADJ, OP_BASE, false, false, c, 0)
                     : all_passes(ctx, 1, OP_BASE, OP_NONE, false, false, c, 0);
  if (!r) r = exchange(ctx, 1);
  int64_t slot = 0;
  int64_t all_pts = 0;
  for (auto& s : ctx->slabs) all_pts += (int64_t)s.nx * ctx->ny * ctx->nk * 2;
  for (int64_t i = 1; i <= nsteps && !r; ++i) {
    const int64_t n = step_offset + i;
    const bool rec = record_stride > 0 && n % record_stride == 0;
    if (!(i == nsteps && defer)) {
      // one fused march: K3(n) and K4(n) (the tail adjoint on the last step)
      r = timed(ctx, all_pts, [&] { return step_fused(ctx, rec, i == nsteps, c, (int)n); });
      if (!r && rec) r = finalize_record(ctx, slot++, false);
      continue;
    }
    // last step with a deferred tail: two passes, the red adjoint left pending
    r = all_passes(ctx, 0, OP_BASE, OP_ADJ, rec, true, c, (int)n);
    if (!r) r = exchange(ctx, 0);
    if (!r) {
      ctx->pending = true;
      ctx->pend_c = c;
    }
  }
  return r;
}

}  // namespace
