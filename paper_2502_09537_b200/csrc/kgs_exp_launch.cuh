// kgs_exp_launch.cuh -- EXPERIMENTAL host dispatch, compiled only with
// -DKGS_EXPERIMENTAL: the fused one-march DP-AVF2 step (ping-pong buffer
// sets, knob "fused_step") and its TMA descriptors.  Included from
// kgs_launch.cuh inside its anonymous namespace.
#pragma once

// fused step: red pieces of one buffer set (StepSmem layout)
constexpr int kStepTY = 8, kStepTK = 32;
using StepS = StepSmem<kStepTY, kStepTK>;

int make_step_maps(kgs_ctx* ctx, const Slab& s, double* red, StepMaps& m) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return fail(ctx, KGS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[4] = {(cuuint64_t)ctx->nk, 4, (cuuint64_t)ctx->ny,
                              (cuuint64_t)(s.nx + 2)};
  const cuuint64_t strides[3] = {(cuuint64_t)ctx->pp * 8, (cuuint64_t)ctx->rs * 8,
                                 (cuuint64_t)ctx->ps * 8};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  const cuuint32_t centre[4] = {kStepTK, 3, kStepTY, 1};
  const cuuint32_t rows2[4] = {kStepTK, 3, 2, 1};
  const cuuint32_t col[4] = {2, 3, kStepTY, 1};
  const cuuint32_t corner[4] = {2, 3, 1, 1};
  CUtensorMap* outs[4] = {&m.centre, &m.rows2, &m.col, &m.corner};
  const cuuint32_t* boxes[4] = {centre, rows2, col, corner};
  for (int i = 0; i < 4; ++i) {
    CUresult r = enc(outs[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, red, dims, strides, boxes[i],
                     es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     promo(ctx->tune_promo_halo), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(ctx, KGS_ECUDA, "cuTensorMapEncodeTiled(step box %d) failed: %d", i, (int)r);
  }
  return KGS_OK;
}

int make_step_maps_for(kgs_ctx* ctx, Slab& s) {
  s.has_smap = false;
  if (s.alt[0] && ctx->ny % kStepTY == 0 && ctx->nk % kStepTK == 0) {
    int r = make_step_maps(ctx, s, s.buf[1], s.smap[0]);
    if (!r) r = make_step_maps(ctx, s, s.alt[1], s.smap[1]);
    if (r) return r;
    s.has_smap = true;
  }
  return KGS_OK;
}

// ---- fused steps (ping-pong buffer sets) ---------------------------------

// Geometry-only test (no allocation): 3-D, tiles divide the planes, and a
// multi-slab run leaves interior K4 planes [1, nx-1).
bool fused_geometry(const kgs_ctx* ctx) {
  if (!ctx->tune_fused || ctx->alt_failed || ctx->d != 3 || ctx->tune_xc < 0) return false;
  if (ctx->ny % kStepTY || ctx->nk % kStepTK) return false;
  for (auto& s : ctx->slabs)
    if (s.nx < 4) return false;
  return true;
}

// Allocate the second buffer set on first use; if it does not fit, run
// two-pass steps from then on (same results, more traffic).
bool fused_ready(kgs_ctx* ctx) {
  if (!fused_geometry(ctx)) return false;
  for (auto& s : ctx->slabs) {
    if (s.alt[0] && s.has_smap) continue;
    if (cudaSetDevice(s.dev) != cudaSuccess) return false;
    const size_t colour_bytes = (size_t)(s.nx + 2) * ctx->ps * sizeof(double);
    for (int c = 0; c < 2 && !ctx->alt_failed; ++c) {
      if (s.alt[c]) continue;
      if (cudaMalloc(&s.alt[c], colour_bytes) != cudaSuccess) {
        cudaGetLastError();
        s.alt[c] = nullptr;
        ctx->alt_failed = true;
      } else {
        s.alt0[c] = s.alt[c] + ctx->ps;
      }
    }
    if (ctx->alt_failed || make_tensor_maps(ctx, s) || !s.has_smap) {
      for (auto& t : ctx->slabs)
        for (int c = 0; c < 2; ++c) {
          if (t.alt[c]) cudaFree(t.alt[c]);
          t.alt[c] = t.alt0[c] = nullptr;
        }
      ctx->alt_failed = true;
      return false;
    }
  }
  return true;
}

void swap_sets(kgs_ctx* ctx) {
  for (auto& s : ctx->slabs) {
    for (int c = 0; c < 2; ++c) {
      std::swap(s.buf[c], s.alt[c]);
      std::swap(s.plane0[c], s.alt0[c]);
    }
    std::swap(s.maps, s.amaps);
    std::swap(s.smap[0], s.smap[1]);
  }
}

template <bool DIAG, int K4OP2, int FORM>
int launch_step_form(kgs_ctx* ctx, Slab& s, const Coeffs& c, int step_no, int xa, int xb) {
  constexpr int NT = kStepTY * kStepTK;
  // FORM 1: step_pass (K4 one plane behind, 4 + 3 slots); FORM 2: step2_pass
  // (K4 two planes behind, 5 + 4 slots, interleaved chains)
  constexpr size_t kBytes = FORM == 1 ? StepS::bytes : Step2Smem<kStepTY, kStepTK, 5, 4>::bytes;
  auto kern = FORM == 1 ? step_pass<DIAG, K4OP2, kStepTY, kStepTK, 2>
                        : step2_pass<DIAG, K4OP2, kStepTY, kStepTK, 2>;
  static int occ_dev[kMaxDevices] = {};
  int& occ = occ_dev[current_device()];
  if (occ == 0) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kBytes));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, kBytes));
    if (occ < 1) return fail(ctx, KGS_ECUDA, "fused step kernel does not fit on an SM");
  }
  StepGeom g{};
  g.rold = s.plane0[1];
  g.bold = s.plane0[0];
  g.rnew = s.alt0[1];
  g.bnew = s.alt0[0];
  g.ps = ctx->ps;
  g.pp = ctx->pp;
  g.rs = ctx->rs;
  g.nx = s.nx;
  g.ny = ctx->ny;
  g.nk = ctx->nk;
  g.x0 = s.x0;
  g.wrap = needs_exchange(ctx) ? 0 : 1;
  g.xa = xa;
  g.xb = xb;
  g.wa = 0;
  g.wb = s.nx;
  g.xc = std::max(1, std::min(ctx->tune_fused_xc, xb - xa));
  g.dbg = ctx->tune_fused_dbg;
  const int64_t ncols = (int64_t)(ctx->ny / kStepTY) * (ctx->nk / kStepTK);
  g.nunits = (int64_t)((xb - xa + g.xc - 1) / g.xc) * ncols;
  const int64_t grid = std::min<int64_t>({g.nunits, (int64_t)occ * ctx->nsm, ctx->grid_cap});
  kern<<<(unsigned)grid, NT, kBytes, s.stream>>>(
      s.smap[0], g, c, s.partials[1] + (int64_t)s.npart[1] * NTERMS, s.bad, step_no);
  ctx->launches++;
  if (DIAG) s.npart[1] += (int)grid;
  CK(cudaGetLastError());
  return KGS_OK;
}

template <bool DIAG, int K4OP2>
int launch_step(kgs_ctx* ctx, Slab& s, const Coeffs& c, int step_no, int xa, int xb) {
  return ctx->tune_fused == 2 ? launch_step_form<DIAG, K4OP2, 2>(ctx, s, c, step_no, xa, xb)
                              : launch_step_form<DIAG, K4OP2, 1>(ctx, s, c, step_no, xa, xb);
}


// One DP-AVF2 step n as a fused march (K3(n) then K4(n), or the red adjoint
// tail when `last`), step-n state in the current set, result in the other;
// the sets are swapped after the launch.  Several slabs: the march does K4
// on planes [1, nx-1) only; the black faces are exchanged and K4 on planes
// 0 and nx-1 runs as a small pass reading the old red (own_in) and the new
// black ghosts, writing the new red; then the red faces are exchanged.
int step_fused(kgs_ctx* ctx, bool rec, bool last, const Coeffs& c, int step_no) {
  const bool multi = needs_exchange(ctx);
  ctx->mirrored[0] = ctx->mirrored[1] = false;  // this path exchanges by copies
  // With fused halo stores this step takes part in their event protocol as
  // one pass k: the ghosts it reads may have been stored by the neighbours'
  // previous pass (wait for their ev_face of k-1), and a later storing pass
  // must wait until this step stopped reading ghosts (ev_face of k below).
  const bool mirror = multi && ctx->mirror && ctx->tune_mirror;
  const int64_t k = ctx->pass_no;
  if (multi) ctx->pass_no++;
  const int ns = (int)ctx->slabs.size();
  for (int i = 0; i < ns; ++i) {
    Slab& s = ctx->slabs[i];
    CK(cudaSetDevice(s.dev));
    if (s.xch_pending) {   // red ghosts of the current set (K3 at planes 0, nx-1)
      CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
      s.xch_pending = false;
    }
    if (mirror && k > 0) {
      CK(cudaStreamWaitEvent(s.stream, ctx->slabs[(i - 1 + ns) % ns].ev_face[(k - 1) & 1], 0));
      CK(cudaStreamWaitEvent(s.stream, ctx->slabs[(i + 1) % ns].ev_face[(k - 1) & 1], 0));
    }
    if (rec) {
      s.npart[1] = 0;
      s.npart[0] = 0;
      if (s.fin_busy[s.pset]) {   // a record reduction still reads this partial set
        CK(cudaStreamWaitEvent(s.stream, s.ev_fin[s.pset], 0));
        s.fin_busy[s.pset] = false;
      }
    }
    const int xa = multi ? 1 : 0, xb = multi ? s.nx - 1 : s.nx;
    int r;
    if (rec) r = last ? launch_step<true, OP_NONE>(ctx, s, c, step_no, xa, xb)
                      : launch_step<true, OP_BASE>(ctx, s, c, step_no, xa, xb);
    else     r = last ? launch_step<false, OP_NONE>(ctx, s, c, step_no, xa, xb)
                      : launch_step<false, OP_BASE>(ctx, s, c, step_no, xa, xb);
    if (r) return r;
  }
  swap_sets(ctx);
  if (!multi) return KGS_OK;
  int r = exchange(ctx, 0);
  const int op2 = last ? OP_NONE : OP_BASE;
  for (auto& s : ctx->slabs) {
    if (r) return r;
    CK(cudaSetDevice(s.dev));
    if (s.xch_pending) {
      CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
      s.xch_pending = false;
    }
    r = launch_pass(ctx, s, 1, OP_ADJ, op2, rec, true, c, step_no, 0, 1, s.alt0[1], nullptr,
                    nullptr);
    if (!r) r = launch_pass(ctx, s, 1, OP_ADJ, op2, rec, true, c, step_no, s.nx - 1, s.nx,
                            s.alt0[1], nullptr, nullptr);
    if (!r && mirror) CK(cudaEventRecord(s.ev_face[k & 1], s.stream));
  }
  if (!r) r = exchange(ctx, 1);
  return r;
}


