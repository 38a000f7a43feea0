// kgs_launch.cuh -- kernel dispatch: simple and marching colour passes (TMA descriptors, tile variants), resident small-grid steps, fused ping-pong steps.
// Part of the single translation unit kgs_host.cu (included in order).
#pragma once

namespace {

// Function attributes (the dynamic shared-memory opt-in) and occupancy are
// per device context: every per-kernel cache below is indexed by the
// current device, so a context whose slabs sit on several GPUs configures
// each of them (the launches set the slab's device first).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}

// ---- kernel dispatch -----------------------------------------------------
// Launch a kernel that opens with griddepcontrol.wait / launch_dependents as
// a programmatic dependent of the previous kernel on the stream (its launch
// and CTA dispatch overlap that kernel's drain), or in plain stream order.
template <typename... KArgs, typename... Args>
cudaError_t launch_dependent(bool pdl, void (*kern)(KArgs...), unsigned grid, unsigned block,
                             size_t smem, cudaStream_t stream, Args... args) {
  if (!pdl) {
    kern<<<grid, block, smem, stream>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int D, int COL, int OP1, int OP2, bool DIAG, bool CHECK>
int launch_t(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c,
             int step_no) {
  auto kern = colour_pass<D, COL, OP1, OP2, DIAG, CHECK>;
  static int occ_dev[kMaxDevices] = {};  // per instantiation and device
  int& occ = occ_dev[current_device()];
  if (occ == 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
    if (occ < 1) occ = 1;
  }
  const int bps = ctx->tune_occ > 0 ? std::min(occ, ctx->tune_occ) : occ;
  int64_t grid = std::min<int64_t>(g.ntiles, (int64_t)bps * ctx->nsm);
  grid = std::min<int64_t>(grid, ctx->grid_cap);
  if (grid < 1) return KGS_OK;  // nothing to do
  double* part = s.partials[COL] + (int64_t)s.npart[COL] * NTERMS;
  CK(launch_dependent(ctx->tune_pdl != 0, kern, (unsigned)grid, kThreads, 0, s.stream, g, c,
                      part, s.bad, step_no));
  ctx->launches++;
  if (DIAG) s.npart[COL] += (int)grid;
  CK(cudaGetLastError());
  return KGS_OK;
}

// ---- TMA descriptors ------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 3-D march kernel variants: tile rows x slots, ring depths, min blocks/SM,
// cluster size, producer warp, rows per thread.  Larger tile cross-sections
// re-read fewer halo rows/slots; deeper rings keep more bytes in flight;
// several rows per thread (RPT) interleave independent fp64 chains, so fewer
// warps (hence more shared memory per CTA for the rings) keep the FP64 pipe
// busy.
template <int TY_, int TK_, int NOTH_, int NOWN_, int MINB_, int CL_ = 1, bool PW_ = false,
          int RPT_ = 1>
struct MarchVariant {
  static constexpr int TY = TY_, TK = TK_, NOTH = NOTH_, NOWN = NOWN_, MINB = MINB_, CL = CL_;
  static constexpr bool PW = PW_;
  static constexpr int RPT = RPT_;
  static constexpr int NT = TY * TK / RPT + (PW ? 32 : 0);   // + the producer warp
  using L = MarchSmem<TY, TK, NOTH, NOWN>;
};
using MV0 = MarchVariant<4, 64, 4, 2, 4>;     // 256 threads, 4 blocks/SM
using MV1 = MarchVariant<8, 64, 4, 2, 2>;     // 512 threads, 2 blocks/SM
using MV2 = MarchVariant<16, 32, 4, 2, 2>;    // 512 threads, 2 blocks/SM
using MV3 = MarchVariant<32, 32, 4, 2, 1>;    // 1024 threads, 1 block/SM
using MV4 = MarchVariant<8, 64, 4, 2, 2, 1, false, 2>;   // 256 threads x 2 rows, 2 blocks/SM
using MV5 = MarchVariant<4, 64, 5, 3, 3, 1, false, 2>;   // 128 threads x 2 rows, deep rings, 3/SM
using MV6 = MarchVariant<4, 64, 4, 2, 4, 1, false, 2>;   // 128 threads x 2 rows, 4 blocks/SM
using MV7 = MarchVariant<16, 64, 4, 2, 1, 1, false, 2>;  // 512 threads x 2 rows, 1 block/SM
using MV8 = MarchVariant<16, 64, 4, 2, 1, 1, false, 4>;  // 256 threads x 4 rows, 1 block/SM
using MV9 = MarchVariant<16, 32, 4, 2, 2, 1, false, 2>;  // 256 threads x 2 rows, 2 blocks/SM
using MV10 = MarchVariant<8, 128, 4, 2, 1, 1, false, 2>; // 512 threads x 2 rows, 1 block/SM
using MV11 = MarchVariant<8, 32, 4, 2, 4, 1, false, 2>;  // 128 threads x 2 rows, 4 blocks/SM
using MV12 = MarchVariant<8, 64, 5, 2, 2, 1, false, 2>;  // MV4 with one more other-colour plane
using MV13 = MarchVariant<4, 64, 4, 2, 4, 8>;  // MV0 in clusters of 8 along y
using MV14 = MarchVariant<4, 64, 4, 2, 4, 4>;  // MV0 in clusters of 4 along y
using MV15 = MarchVariant<4, 64, 4, 2, 4, 1, true>;  // MV0 + a producer warp, no block barrier
constexpr int kMarchVariants = kMarchVariantSlots;
#define KGS_MV_LIST(F) F(MV0), F(MV1), F(MV2), F(MV3), F(MV4), F(MV5), F(MV6), F(MV7), F(MV8), \
                       F(MV9), F(MV10), F(MV11), F(MV12), F(MV13), F(MV14), F(MV15)
// Variants compiled into this build: the default library carries MV4 (the
// default), MV0 (one point per thread, the round-1 kernel) and MV1 (8 x 64,
// one point per thread); every other shape was measured slower (DESIGN.md
// §5) and exists only in -DKGS_EXPERIMENTAL builds.
#ifdef KGS_EXPERIMENTAL
constexpr bool kVarBuilt[kMarchVariants] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
#else
constexpr bool kVarBuilt[kMarchVariants] = {1, 1, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
#define KGS_MV_TY(V) V::TY
#define KGS_MV_TK(V) V::TK
#define KGS_MV_CL(V) V::CL
constexpr int kVarTY[kMarchVariants] = {KGS_MV_LIST(KGS_MV_TY)};
constexpr int kVarTK[kMarchVariants] = {KGS_MV_LIST(KGS_MV_TK)};
constexpr int kVarCL[kMarchVariants] = {KGS_MV_LIST(KGS_MV_CL)};
#undef KGS_MV_TY
#undef KGS_MV_TK
#undef KGS_MV_CL

// L2 sector promotion of the TMA boxes.  The two-slot halo columns are 16 B
// inside a neighbouring tile's lines: promoting them to 256-B fetches would
// pull whole blocks of that tile from HBM.
CUtensorMapL2promotion promo(int v) {
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// 4-D view of one colour array with dims ordered (slot, field, row, plane)
// -- strides 8, pp*8, nk*8, ps*8 bytes -- so that a box lands in shared
// memory as [row][field][slot] (MarchSmem); per variant four box shapes.
int make_maps_for(kgs_ctx* ctx, Slab& s, double* const bufs[2],
                  MarchMaps (&maps)[kMarchVariantSlots][2]) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return fail(ctx, KGS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[4] = {(cuuint64_t)ctx->nk, 4, (cuuint64_t)ctx->ny,
                              (cuuint64_t)(s.nx + 2)};
  const cuuint64_t strides[3] = {(cuuint64_t)ctx->pp * 8, (cuuint64_t)ctx->rs * 8,
                                 (cuuint64_t)ctx->ps * 8};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  for (int v = 0; v < kMarchVariants; ++v) {
    const int ty = kVarTY[v], tk = kVarTK[v];
    s.has_tmaps[v] = kVarBuilt[v] && ctx->d == 3 && ctx->ny % (ty * kVarCL[v]) == 0 &&
                     ctx->nk % tk == 0 && ctx->nk >= 2 && (ctx->rs * 8) % 16 == 0;
    if (!s.has_tmaps[v]) continue;
    const cuuint32_t centre[4] = {(cuuint32_t)tk, 3, (cuuint32_t)ty, 1};
    const cuuint32_t row[4] = {(cuuint32_t)tk, 3, 1, 1};
    const cuuint32_t col[4] = {2, 3, (cuuint32_t)ty, 1};
    const cuuint32_t own[4] = {(cuuint32_t)tk, 4, (cuuint32_t)ty, 1};
    for (int c = 0; c < 2; ++c) {
      MarchMaps& m = maps[v][c];
      CUtensorMap* outs[4] = {&m.centre, &m.row, &m.col, &m.own};
      const cuuint32_t* boxes[4] = {centre, row, col, own};
      for (int i = 0; i < 4; ++i) {
        CUresult r = enc(outs[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, bufs[c], dims, strides,
                         boxes[i], es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         promo(i == 3 ? ctx->tune_promo_tile : ctx->tune_promo_halo),
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
          return fail(ctx, KGS_ECUDA, "cuTensorMapEncodeTiled(variant %d, box %d) failed: %d", v,
                      i, (int)r);
      }
    }
  }
  return KGS_OK;
}

#ifdef KGS_EXPERIMENTAL
int make_step_maps_for(kgs_ctx* ctx, Slab& s);
#endif

int make_tensor_maps(kgs_ctx* ctx, Slab& s) {
  int r = make_maps_for(ctx, s, s.buf, s.maps);
  if (!r && s.alt[0]) r = make_maps_for(ctx, s, s.alt, s.amaps);
#ifdef KGS_EXPERIMENTAL
  if (!r) r = make_step_maps_for(ctx, s);
#endif
  return r;
}

template <typename Var, int COL, int OP1, int OP2, bool DIAG, bool CHECK, int DBG = 0,
          int GF = 2>
int launch_march(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c, int step_no,
                 int v) {
  using L = typename Var::L;
  constexpr int CL = Var::CL;
  // record passes carry 8 more accumulators: one-point-per-thread variants
  // give them half the blocks per SM (more registers, no spills); the
  // two-rows-per-thread variants already run few, wide blocks and keep them
  constexpr int kMinB = (DIAG && Var::RPT == 1) ? (Var::MINB > 1 ? Var::MINB / 2 : 1) : Var::MINB;
  auto kern = march_pass<COL, OP1, OP2, DIAG, CHECK, Var::TY, Var::TK, Var::NOTH, Var::NOWN,
                         kMinB, DBG, CL, Var::PW, Var::RPT, GF>;
  // resident CTAs per SM (or clusters per GPU / nsm when CL > 1), per device
  static int occ_dev[kMaxDevices] = {};
  static int max_clusters_dev[kMaxDevices] = {};
  const int dev = current_device();
  int& occ = occ_dev[dev];
  int& max_clusters = max_clusters_dev[dev];
  if (occ == 0) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Var::NT, L::bytes));
    if (occ < 1) return fail(ctx, KGS_ECUDA, "march kernel does not fit on an SM");
    if (CL > 1) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(CL * 64);
      cfg.blockDim = dim3(Var::NT);
      cfg.dynamicSmemBytes = L::bytes;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg));
      if (max_clusters < 1) return fail(ctx, KGS_ECUDA, "march cluster does not fit");
    }
  }
  const int bps = ctx->tune_occ > 0 ? std::min(occ, ctx->tune_occ) : occ;
  const int sms = ctx->tune_sms > 0 ? std::min(ctx->nsm, ctx->tune_sms) : ctx->nsm;
  int64_t G = std::min<int64_t>((int64_t)bps * sms, ctx->grid_cap);
  if (CL > 1) G = std::min<int64_t>(G, (int64_t)max_clusters * CL) / CL * CL;
  const int64_t cols = (int64_t)(g.ny / Var::TY) * (g.nk / Var::TK);
  const int nxr = g.xb - g.xa;
  MarchCfg mc;
  // wave barriers (knob march_wave_sync, default on): one slab per device
  // only (concurrent grids of other slabs or of the pipeline's transfers on
  // the same GPU would keep CTAs of this one from being resident)
  bool shared_dev = ctx->in_pipeline;
  for (auto& t : ctx->slabs) shared_dev = shared_dev || (&t != &s && t.dev == s.dev);
  mc.wsync = (ctx->tune_wsync && CL == 1 && !Var::PW && !shared_dev) ? 1 : 0;
  if (ctx->tune_xc > 0) mc.xc = std::min(ctx->tune_xc, nxr);
  else if (mc.wsync)  // 256-plane units: drift reset every wave, few barriers
    mc.xc = std::min(nxr, 256);
  else  // ~8 units per resident block for load balance, >= 8 planes per unit
    mc.xc = (int)std::max<int64_t>(std::min<int64_t>(nxr, 8),
                                   std::min<int64_t>(nxr, (int64_t)nxr * cols / (8 * G)));
  mc.nunits = (int64_t)((nxr + mc.xc - 1) / mc.xc) * cols;
  mc.sync = std::max(1, ctx->tune_sync);
  const int64_t grid = std::min<int64_t>(mc.nunits, G) / CL * CL;
  if (grid < 1) return KGS_OK;
  // wave barriers: arrivals after waves 0 .. W-2
  mc.wctr = s.wctr;
  mc.wbase = s.wbase;
  if (mc.wsync) {
    const int64_t waves = (mc.nunits + grid - 1) / grid;
    if (waves > 1) s.wbase += (unsigned long long)((waves - 1) * grid);
  }

  if (CL > 1) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(Var::NT);
    cfg.dynamicSmemBytes = L::bytes;
    cfg.stream = s.stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, s.maps[v][COL ^ 1], s.maps[v][COL], g, c,
                          s.partials[COL] + (int64_t)s.npart[COL] * NTERMS, s.bad, step_no,
                          mc));
  } else {
    CK(launch_dependent(ctx->tune_pdl != 0, kern, (unsigned)grid, (unsigned)Var::NT, L::bytes,
                        s.stream, s.maps[v][COL ^ 1], s.maps[v][COL], g, c,
                        s.partials[COL] + (int64_t)s.npart[COL] * NTERMS, s.bad, step_no, mc));
  }
  ctx->launches++;
  if (DIAG) s.npart[COL] += (int)grid;
  CK(cudaGetLastError());
  return KGS_OK;
}

// ---- resident steps (whole state in one CTA's shared memory) -------------
constexpr size_t kResidentMaxBytes = 200 * 1024;

bool resident_eligible(const kgs_ctx* ctx) {
  if (!ctx->tune_resident || ctx->slabs.size() != 1 || needs_exchange(ctx))
    return false;
  const Slab& s = ctx->slabs[0];
  return (size_t)s.nx * ctx->ps * 2 * sizeof(double) <= kResidentMaxBytes;
}

template <int D>
int launch_resident_d(kgs_ctx* ctx, Slab& s, const Coeffs& c, const ResidentCfg& rc) {
  auto kern = resident_steps<D>;
  static bool attr_dev[kMaxDevices] = {};
  bool& attr = attr_dev[current_device()];
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kResidentMaxBytes));
    attr = true;
  }
  PassGeom gb = make_geom(ctx, s, 0, 0, s.nx), gr = make_geom(ctx, s, 1, 0, s.nx);
  const size_t bytes = (size_t)s.nx * ctx->ps * 2 * sizeof(double);
  kern<<<1, 1024, bytes, s.stream>>>(gb, gr, c, rc, s.records, s.bad);
  ctx->launches++;
  CK(cudaGetLastError());
  return KGS_OK;
}

int launch_resident(kgs_ctx* ctx, const Coeffs& c, int64_t nsteps, int64_t step_offset,
                    int64_t record_stride, bool head_fused, bool defer) {
  Slab& s = ctx->slabs[0];
  CK(cudaSetDevice(s.dev));
  ResidentCfg rc;
  rc.nsteps = nsteps;
  rc.step_offset = step_offset;
  rc.record_stride = record_stride;
  rc.head_fused = head_fused ? 1 : 0;
  rc.defer = defer ? 1 : 0;
  switch (ctx->d) {
    case 1: return launch_resident_d<1>(ctx, s, c, rc);
    case 2: return launch_resident_d<2>(ctx, s, c, rc);
    default: return launch_resident_d<3>(ctx, s, c, rc);
  }
}

int exchange(kgs_ctx* ctx, int col);
int launch_pass(kgs_ctx* ctx, Slab& s, int col, int op1, int op2, bool diag,
                bool check, const Coeffs& c, int step_no, int xa, int xb,
                const double* own_in, double* mir_lo, double* mir_hi);
#ifdef KGS_EXPERIMENTAL
#include "kgs_exp_launch.cuh"
#endif

// march variant to use for this pass, or -1 for the simple kernel
int march_variant(const kgs_ctx* ctx, const Slab& s, const PassGeom& g) {
  if (ctx->d != 3 || ctx->tune_xc < 0 || g.xb - g.xa < 1) return -1;
  if (g.own != g.own_out) return -1;  // reads another buffer: simple kernel
  int v = ctx->tune_variant;
  if (v >= 0 && v < kMarchVariants && s.has_tmaps[v]) return v;
  for (v = 0; v < kMarchVariants; ++v)   // fall back to any eligible variant
    if (s.has_tmaps[v]) return v;
  return -1;
}

template <int COL, int O1, int O2, bool DG, bool CH, int GF>
int launch_march_gf(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c, int step_no,
                    int v) {
  switch (v) {
#define KGS_MV_CASE(N) \
    case N: return launch_march<MV##N, COL, O1, O2, DG, CH, 0, GF>(ctx, s, g, c, step_no, v);
    KGS_MV_CASE(0) KGS_MV_CASE(1)
#ifdef KGS_EXPERIMENTAL
    KGS_MV_CASE(2) KGS_MV_CASE(3) KGS_MV_CASE(5) KGS_MV_CASE(6) KGS_MV_CASE(7) KGS_MV_CASE(8)
    KGS_MV_CASE(9) KGS_MV_CASE(10) KGS_MV_CASE(11) KGS_MV_CASE(12) KGS_MV_CASE(13)
    KGS_MV_CASE(14) KGS_MV_CASE(15)
#endif
#undef KGS_MV_CASE
    default: return launch_march<MV4, COL, O1, O2, DG, CH, 0, GF>(ctx, s, g, c, step_no, v);
  }
}

template <int COL, int O1, int O2, bool DG, bool CH>
int launch_march_any(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c, int step_no,
                     int v) {
  // record passes of the red colour: the gradient-term form (knob record_form)
  if constexpr (DG && COL == 1) {
    if (ctx->tune_gform == 1)
      return launch_march_gf<COL, O1, O2, DG, CH, 1>(ctx, s, g, c, step_no, v);
  }
  return launch_march_gf<COL, O1, O2, DG, CH, 2>(ctx, s, g, c, step_no, v);
}

template <int D, int COL>
int launch_col(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c,
               int op1, int op2, bool diag, bool check, int step_no) {
#define KGS_CASE(O1, O2, DG, CH)                                          \
  if (op1 == O1 && op2 == O2 && diag == DG && check == CH) {             \
    if (D == 3) {                                                        \
      const int v_ = march_variant(ctx, s, g);                           \
      if (v_ >= 0)                                                       \
        return launch_march_any<COL, O1, O2, DG, CH>(ctx, s, g, c, step_no, v_); \
    }                                                                    \
    return launch_t<D, COL, O1, O2, DG, CH>(ctx, s, g, c, step_no);      \
  }
  // single sweeps (kgs_sweep, head)
  KGS_CASE(OP_BASE, OP_NONE, false, false)
  KGS_CASE(OP_ADJ, OP_NONE, false, false)
  // diagnostics / finiteness only
  KGS_CASE(OP_NONE, OP_NONE, true, false)
  KGS_CASE(OP_NONE, OP_NONE, false, true)
  if (COL == 0) {  // K3: black base(n) + adjoint(n)
    KGS_CASE(OP_BASE, OP_ADJ, false, true)
    KGS_CASE(OP_BASE, OP_ADJ, true, true)
  } else {  // K4: red adjoint(n) + base(n+1); tail: red adjoint(n)
    KGS_CASE(OP_ADJ, OP_BASE, false, false)   // deferred tail fused into a head
    KGS_CASE(OP_ADJ, OP_BASE, false, true)
    KGS_CASE(OP_ADJ, OP_BASE, true, true)
    KGS_CASE(OP_ADJ, OP_NONE, false, true)
    KGS_CASE(OP_ADJ, OP_NONE, true, true)
  }
#undef KGS_CASE
  return fail(ctx, KGS_EINVAL, "unsupported pass combination %d/%d/%d/%d",
              op1, op2, (int)diag, (int)check);
}

// own_in: read this colour from another buffer (same geometry) and write
// the result to the current one; uses the simple kernel.
int launch_pass(kgs_ctx* ctx, Slab& s, int col, int op1, int op2, bool diag,
                bool check, const Coeffs& c, int step_no, int xa = 0, int xb = -1,
                const double* own_in = nullptr, double* mir_lo = nullptr,
                double* mir_hi = nullptr) {
  PassGeom g = make_geom(ctx, s, col, xa, xb < 0 ? s.nx : xb);
  if (own_in) g.own = const_cast<double*>(own_in);
  g.mir_lo = mir_lo;
  g.mir_hi = mir_hi;
  switch (ctx->d * 2 + col) {
    case 2: return launch_col<1, 0>(ctx, s, g, c, op1, op2, diag, check, step_no);
    case 3: return launch_col<1, 1>(ctx, s, g, c, op1, op2, diag, check, step_no);
    case 4: return launch_col<2, 0>(ctx, s, g, c, op1, op2, diag, check, step_no);
    case 5: return launch_col<2, 1>(ctx, s, g, c, op1, op2, diag, check, step_no);
    case 6: return launch_col<3, 0>(ctx, s, g, c, op1, op2, diag, check, step_no);
    case 7: return launch_col<3, 1>(ctx, s, g, c, op1, op2, diag, check, step_no);
  }
  return fail(ctx, KGS_EINVAL, "bad dimension %d", ctx->d);
}

}  // namespace
