// kgs_host.cu -- C ABI (include/kgs_b200.h) over the sm_100a colour-pass
// kernels: contexts, slabs, halo exchange, fused DP-AVF2 stepping loop,
// diagnostics.  See DESIGN.md for the pass schedule and the roofline.
#include "../../include/kgs_b200.h"
#include "kgs_device.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace kgs;

namespace {

thread_local std::string g_last_error = "no error";

// ---- NCCL, loaded lazily so single-GPU use never needs it --------------
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool load_nccl(std::string& err) {
  if (g_nccl.tried) {
    if (!g_nccl.ok) err = "libnccl.so.2 could not be loaded";
    return g_nccl.ok;
  }
  g_nccl.tried = true;
  // RTLD_NOLOAD first: reuse the NCCL torch already mapped into the process.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return false;
  }
#define KGS_SYM(field, name)                                         \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) { err = "missing NCCL symbol " name; return false; }
  KGS_SYM(GetUniqueId, "ncclGetUniqueId");
  KGS_SYM(CommInitRank, "ncclCommInitRank");
  KGS_SYM(CommDestroy, "ncclCommDestroy");
  KGS_SYM(Send, "ncclSend");
  KGS_SYM(Recv, "ncclRecv");
  KGS_SYM(GroupStart, "ncclGroupStart");
  KGS_SYM(GroupEnd, "ncclGroupEnd");
  KGS_SYM(GetErrorString, "ncclGetErrorString");
#undef KGS_SYM
  g_nccl.ok = true;
  return true;
}

struct Slab {
  int dev = 0;
  int64_t x0 = 0;  // global first plane
  int nx = 0;      // planes
  double* buf[2] = {nullptr, nullptr};    // colour c, ghost plane -1
  double* plane0[2] = {nullptr, nullptr}; // colour c, element (x=0,f=0,y=0,k=0)
  MarchMaps maps[6][2];  // [march variant][colour]: TMA descriptors
  bool has_tmaps[6] = {};  // variant fits this geometry
  // fused steps (ping-pong): the other buffer set and its descriptors
  double* alt[2] = {nullptr, nullptr};
  double* alt0[2] = {nullptr, nullptr};
  MarchMaps amaps[6][2];
  StepMaps smap[2];        // red of [0] the current set, [1] the other set
  bool has_smap = false;
  double* partials[2] = {nullptr, nullptr};  // per colour pass, grid * NTERMS
  int npart[2] = {0, 0};                     // blocks that wrote partials
  double* records = nullptr;                 // device [cap * NTERMS]
  int64_t rec_cap = 0;
  unsigned long long* bad = nullptr;
  double* stage = nullptr;  // natural-layout staging planes
  int stage_planes = 0;
  cudaStream_t stream = nullptr;    // compute
  cudaStream_t cstream = nullptr;   // halo exchange (copies / NCCL)
  cudaEvent_t ev_done = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
  cudaEvent_t ev_bnd = nullptr;     // boundary planes of the last pass written
  cudaEvent_t ev_xch = nullptr;     // last exchange into this slab's ghosts done
  bool xch_pending = false;
  cudaEvent_t ev_face[2] = {nullptr, nullptr};  // boundary planes of pass k written (k & 1)
  // pipelined host integration (kgs_integrate_host)
  cudaStream_t dstream = nullptr;   // downloads
  double* pipe_up = nullptr;        // natural-layout staging, one chunk of 4 fields
  double* pipe_dn = nullptr;
  int64_t pipe_stage = 0;           // doubles per staging buffer
  double* pipe_part = nullptr;      // per-record DIAG partials
  int64_t pipe_part_cap = 0;
  std::vector<cudaEvent_t> pipe_ev; // arrival / final events per chunk
};

}  // namespace

struct kgs_ctx {
  int d = 3;
  int64_t N = 0;
  double a = 0, b = 1, h = 1;
  int ny = 1, nk = 1, nz = 1;   // rows per plane, slots per row, natural row
  int64_t nxg = 1;              // global planes
  int rs = 0;                   // row stride (nk)
  int64_t pp = 0, ps = 0;       // field stride in a plane (ny*nk), plane stride
  std::vector<Slab> slabs;
  bool dist = false;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  std::string err = "no error";
  int64_t launches = 0;
  double last_ms = 0.0;
  int nsm = 148;
  int grid_cap = 0;  // max persistent grid (blocks), sizes partials
  // tuning knobs (kgs_set_tuning): rows per tile, band height, blocks/SM cap
  int tune_ty = 4, tune_band_rows = 64, tune_occ = 0;
  int tune_xc = 0;  // march kernel planes per unit (0 auto, < 0 disables it)
  int tune_variant = 0;  // march kernel tile variant (MV0..MV3)
  int tune_promo_halo = 0, tune_promo_tile = 0;  // TMA L2 promotion (0 none .. 3 256B)
  int tune_sync = 4;     // march clusters: planes between cluster barriers
  // deferred tail (KGS_STEP_DEFER_TAIL): the red adjoint of the last step is
  // pending and fuses with the next call's head when the coefficients match
  bool pending = false;
  Coeffs pend_c{};
  int tune_fused = 0;      // fused one-march DP-AVF2 steps (opt-in until faster)
  int tune_fused_xc = 128; // fused step: K4 planes per unit
  int tune_fused_dbg = 0;  // fused step timing experiments (results invalid)
  int tune_resident = 1;   // small grids: whole call in one launch (shared memory)
  int tune_tstore = 2;
  int tune_pipe = 1;         // kgs_integrate_host: overlap upload | passes | download
  int tune_pipe_chunk = 32;  // planes per transfer chunk     // march own-tile write: 0 STG, 1 TMA bulk store, 2 + L2 evict-first
  // fused halo exchange (single-process slabs): boundary launches
  // store their faces straight into the neighbours' ghost planes
  bool mirror = false;       // possible for this context (peer-accessible neighbours)
  int tune_mirror = 1;       // knob "mirror_halo"
  int64_t pass_no = 0;       // colour passes issued with the interior/boundary split
  bool mirrored[2] = {false, false};  // faces of colour c already in the ghosts
  bool alt_failed = false; // the second buffer set did not fit: two-pass steps
  int64_t timed_pts = 0;   // points updated twice per timed launch
  // per-pass timing (slab 0's stream): event pairs around fused passes
  bool pass_timing = false;
  std::vector<cudaEvent_t> pass_ev;
  size_t pass_ev_used = 0;
  int64_t pass_count = 0;
  double pass_ms = 0.0;
};

namespace {

int fail(kgs_ctx* c, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  g_last_error = buf;
  return code;
}

#define CK(call)                                                          \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess)                                                \
      return fail(ctx, KGS_ECUDA, "%s failed: %s (%s:%d)", #call,         \
                  cudaGetErrorString(e_), __FILE__, __LINE__);            \
  } while (0)

#define NK(call)                                                          \
  do {                                                                    \
    ncclResult_t r_ = (call);                                             \
    if (r_ != ncclSuccess)                                                \
      return fail(ctx, KGS_ENCCL, "%s failed: %s", #call,                 \
                  g_nccl.GetErrorString(r_));                             \
  } while (0)

// ---- tile geometry -------------------------------------------------------
constexpr int kThreads = 256;

int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

PassGeom make_geom(const kgs_ctx* ctx, const Slab& s, int col, int xa, int xb) {
  PassGeom g{};
  g.own = s.plane0[col];
  g.own_out = g.own;
  g.mir_lo = g.mir_hi = nullptr;
  g.tstore = ctx->tune_tstore;
  g.oth = s.plane0[col ^ 1];
  g.ps = ctx->ps;
  g.pp = ctx->pp;
  g.rs = ctx->rs;
  g.nx = s.nx;
  g.ny = ctx->ny;
  g.nk = ctx->nk;
  g.xa = xa;
  g.xb = xb;
  g.x0 = s.x0;
  g.wrap = (ctx->slabs.size() == 1 && !(ctx->dist && ctx->nranks > 1)) ? 1 : 0;
  // 3-D: tk slots x ty rows (rows y+-1 shared through L1 inside the tile);
  // otherwise one row segment of up to 256 slots.
  int tk = std::min(kThreads, pow2ceil(ctx->nk));
  if (ctx->d == 3) tk = std::min(tk, kThreads / std::max(1, ctx->tune_ty));
  int ty = std::min(kThreads / tk, pow2ceil(ctx->ny));
  g.tk = tk;
  g.ty = ty;
  g.nkt = (ctx->nk + tk - 1) / tk;
  g.nyt = (ctx->ny + ty - 1) / ty;
  // y-bands: tiles are visited band by band, and inside a band plane by
  // plane, so the other colour's planes x-1, x, x+1 of a band are re-read
  // from L2 a few hundred tiles apart instead of a whole plane apart.
  int target = std::max(1, ctx->tune_band_rows / ty);
  int nbt = 1;
  for (int v = 1; v <= std::min(target, g.nyt); ++v)
    if (g.nyt % v == 0) nbt = v;
  if (ctx->tune_band_rows <= 0) nbt = g.nyt;  // no banding
  g.nbt = nbt;
  g.ntiles = (int64_t)(xb - xa) * g.nyt * g.nkt;
  return g;
}

// ---- kernel dispatch -----------------------------------------------------
template <int D, int COL, int OP1, int OP2, bool DIAG, bool CHECK>
int launch_t(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c,
             int step_no) {
  auto kern = colour_pass<D, COL, OP1, OP2, DIAG, CHECK>;
  static int occ = 0;  // per instantiation; all devices are B200
  if (occ == 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
    if (occ < 1) occ = 1;
  }
  const int bps = ctx->tune_occ > 0 ? std::min(occ, ctx->tune_occ) : occ;
  int64_t grid = std::min<int64_t>(g.ntiles, (int64_t)bps * ctx->nsm);
  grid = std::min<int64_t>(grid, ctx->grid_cap);
  if (grid < 1) return KGS_OK;  // nothing to do
  kern<<<(unsigned)grid, kThreads, 0, s.stream>>>(
      g, c, s.partials[COL] + (int64_t)s.npart[COL] * NTERMS, s.bad, step_no);
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

// 3-D march kernel variants: tile rows x slots, ring depths, min blocks/SM.
// Larger tile cross-sections re-read fewer halo rows/slots.
template <int TY_, int TK_, int NOTH_, int NOWN_, int MINB_, int CL_ = 1>
struct MarchVariant {
  static constexpr int TY = TY_, TK = TK_, NOTH = NOTH_, NOWN = NOWN_, MINB = MINB_, CL = CL_;
  static constexpr int NT = TY * TK;
  using L = MarchSmem<TY, TK, NOTH, NOWN>;
};
using MV0 = MarchVariant<4, 64, 4, 2, 4>;     // 256 threads, 4 blocks/SM
using MV1 = MarchVariant<8, 64, 4, 2, 2>;     // 512 threads, 2 blocks/SM
using MV2 = MarchVariant<16, 32, 4, 2, 2>;    // 512 threads, 2 blocks/SM
using MV3 = MarchVariant<32, 32, 4, 2, 1>;    // 1024 threads, 1 block/SM
using MV4 = MarchVariant<4, 64, 4, 2, 4, 8>;  // MV0 in clusters of 8 along y
using MV5 = MarchVariant<4, 64, 4, 2, 4, 4>;  // MV0 in clusters of 4 along y
constexpr int kMarchVariants = 6;
constexpr int kVarTY[kMarchVariants] = {MV0::TY, MV1::TY, MV2::TY, MV3::TY, MV4::TY, MV5::TY};
constexpr int kVarTK[kMarchVariants] = {MV0::TK, MV1::TK, MV2::TK, MV3::TK, MV4::TK, MV5::TK};
constexpr int kVarCL[kMarchVariants] = {MV0::CL, MV1::CL, MV2::CL, MV3::CL, MV4::CL, MV5::CL};

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
int make_maps_for(kgs_ctx* ctx, Slab& s, double* const bufs[2], MarchMaps (&maps)[6][2]) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return fail(ctx, KGS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[4] = {(cuuint64_t)ctx->nk, 4, (cuuint64_t)ctx->ny,
                              (cuuint64_t)(s.nx + 2)};
  const cuuint64_t strides[3] = {(cuuint64_t)ctx->pp * 8, (cuuint64_t)ctx->rs * 8,
                                 (cuuint64_t)ctx->ps * 8};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  for (int v = 0; v < kMarchVariants; ++v) {
    const int ty = kVarTY[v], tk = kVarTK[v];
    s.has_tmaps[v] = ctx->d == 3 && ctx->ny % (ty * kVarCL[v]) == 0 && ctx->nk % tk == 0 &&
                     ctx->nk >= 2 && (ctx->rs * 8) % 16 == 0;
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

// fused step: red pieces of one buffer set (StepSmem layout)
constexpr int kStepTY = 16, kStepTK = 32;
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

int make_tensor_maps(kgs_ctx* ctx, Slab& s) {
  int r = make_maps_for(ctx, s, s.buf, s.maps);
  if (!r && s.alt[0]) r = make_maps_for(ctx, s, s.alt, s.amaps);
  s.has_smap = false;
  if (!r && s.alt[0] && ctx->ny % kStepTY == 0 && ctx->nk % kStepTK == 0) {
    r = make_step_maps(ctx, s, s.buf[1], s.smap[0]);
    if (!r) r = make_step_maps(ctx, s, s.alt[1], s.smap[1]);
    if (!r) s.has_smap = true;
  }
  return r;
}

template <typename Var, int COL, int OP1, int OP2, bool DIAG, bool CHECK, int DBG = 0>
int launch_march(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c, int step_no,
                 int v) {
  using L = typename Var::L;
  constexpr int CL = Var::CL;
  auto kern = march_pass<COL, OP1, OP2, DIAG, CHECK, Var::TY, Var::TK, Var::NOTH, Var::NOWN,
                         DIAG ? (Var::MINB > 1 ? Var::MINB / 2 : 1) : Var::MINB, DBG, CL>;
  static int occ = 0;  // resident CTAs per SM (or clusters per GPU / nsm when CL > 1)
  static int max_clusters = 0;
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
  int64_t G = std::min<int64_t>((int64_t)bps * ctx->nsm, ctx->grid_cap);
  if (CL > 1) G = std::min<int64_t>(G, (int64_t)max_clusters * CL) / CL * CL;
  const int64_t cols = (int64_t)(g.ny / Var::TY) * (g.nk / Var::TK);
  const int nxr = g.xb - g.xa;
  MarchCfg mc;
  if (ctx->tune_xc > 0) mc.xc = std::min(ctx->tune_xc, nxr);
  else  // ~8 units per resident block for load balance, >= 8 planes per unit
    mc.xc = (int)std::max<int64_t>(std::min<int64_t>(nxr, 8),
                                   std::min<int64_t>(nxr, (int64_t)nxr * cols / (8 * G)));
  mc.nunits = (int64_t)((nxr + mc.xc - 1) / mc.xc) * cols;
  mc.sync = std::max(1, ctx->tune_sync);
  const int64_t grid = std::min<int64_t>(mc.nunits, G) / CL * CL;
  if (grid < 1) return KGS_OK;
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
    kern<<<(unsigned)grid, Var::NT, L::bytes, s.stream>>>(
        s.maps[v][COL ^ 1], s.maps[v][COL], g, c,
        s.partials[COL] + (int64_t)s.npart[COL] * NTERMS, s.bad, step_no, mc);
  }
  ctx->launches++;
  if (DIAG) s.npart[COL] += (int)grid;
  CK(cudaGetLastError());
  return KGS_OK;
}

// ---- resident steps (whole state in one CTA's shared memory) -------------
constexpr size_t kResidentMaxBytes = 200 * 1024;

bool resident_eligible(const kgs_ctx* ctx) {
  if (!ctx->tune_resident || ctx->slabs.size() != 1 || (ctx->dist && ctx->nranks > 1))
    return false;
  const Slab& s = ctx->slabs[0];
  return (size_t)s.nx * ctx->ps * 2 * sizeof(double) <= kResidentMaxBytes;
}

template <int D>
int launch_resident_d(kgs_ctx* ctx, Slab& s, const Coeffs& c, const ResidentCfg& rc) {
  auto kern = resident_steps<D>;
  static bool attr = false;
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

// ---- fused steps (ping-pong buffer sets) ---------------------------------
bool needs_exchange(const kgs_ctx* ctx);
int exchange(kgs_ctx* ctx, int col);

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

template <bool DIAG, int K4OP2>
int launch_step(kgs_ctx* ctx, Slab& s, const Coeffs& c, int step_no, int xa, int xb) {
  constexpr int NT = kStepTY * kStepTK;
  auto kern = step_pass<DIAG, K4OP2, kStepTY, kStepTK, 2>;
  static int occ = 0;
  if (occ == 0) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)StepS::bytes));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, StepS::bytes));
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
  kern<<<(unsigned)grid, NT, StepS::bytes, s.stream>>>(
      s.smap[0], g, c, s.partials[1] + (int64_t)s.npart[1] * NTERMS, s.bad, step_no);
  ctx->launches++;
  if (DIAG) s.npart[1] += (int)grid;
  CK(cudaGetLastError());
  return KGS_OK;
}

int launch_pass(kgs_ctx* ctx, Slab& s, int col, int op1, int op2, bool diag,
                bool check, const Coeffs& c, int step_no, int xa, int xb,
                const double* own_in, double* mir_lo, double* mir_hi);

// One DP-AVF2 step n as a fused march (K3(n) then K4(n), or the red adjoint
// tail when `last`), step-n state in the current set, result in the other;
// the sets are swapped after the launch.  Several slabs: the march does K4
// on planes [1, nx-1) only; the black faces are exchanged and K4 on planes
// 0 and nx-1 runs as a small pass reading the old red (own_in) and the new
// black ghosts, writing the new red; then the red faces are exchanged.
int step_fused(kgs_ctx* ctx, bool rec, bool last, const Coeffs& c, int step_no) {
  const bool multi = needs_exchange(ctx);
  ctx->mirrored[0] = ctx->mirrored[1] = false;  // this path exchanges by copies
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    if (s.xch_pending) {   // red ghosts of the current set (K3 at planes 0, nx-1)
      CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
      s.xch_pending = false;
    }
    if (rec) { s.npart[1] = 0; s.npart[0] = 0; }
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
  }
  if (!r) r = exchange(ctx, 1);
  return r;
}

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

template <int COL, int O1, int O2, bool DG, bool CH>
int launch_march_any(kgs_ctx* ctx, Slab& s, const PassGeom& g, const Coeffs& c, int step_no,
                     int v) {
  switch (v) {
    case 0: return launch_march<MV0, COL, O1, O2, DG, CH>(ctx, s, g, c, step_no, v);
    case 1: return launch_march<MV1, COL, O1, O2, DG, CH>(ctx, s, g, c, step_no, v);
    case 2: return launch_march<MV2, COL, O1, O2, DG, CH>(ctx, s, g, c, step_no, v);
    case 3: return launch_march<MV3, COL, O1, O2, DG, CH>(ctx, s, g, c, step_no, v);
    case 4: return launch_march<MV4, COL, O1, O2, DG, CH>(ctx, s, g, c, step_no, v);
    default: return launch_march<MV5, COL, O1, O2, DG, CH>(ctx, s, g, c, step_no, v);
  }
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

// ---- halo exchange of colour `col` faces (P, Q, U of planes 0 and nx-1) --
// The three fields of a plane are contiguous ([P|Q|U|V] per plane), so a
// face is ONE contiguous run of 3*pp doubles.
bool needs_exchange(const kgs_ctx* ctx) {
  return ctx->dist ? ctx->nranks > 1 : ctx->slabs.size() > 1;
}

// Start the exchange of colour `col` faces (P, Q, U of planes 0 and nx-1)
// on each slab's comm stream, after the boundary planes of the pass that
// wrote them (ev_bnd); completion is ev_xch, which the next pass waits for
// only before ITS boundary planes -- the interior planes overlap the
// transfer.  The three fields of a plane are contiguous ([P|Q|U|V] per
// plane), so a face is ONE contiguous run of 3*pp doubles.
int exchange(kgs_ctx* ctx, int col) {
  if (!needs_exchange(ctx)) return KGS_OK;  // a single slab wraps in the kernel
  if (ctx->mirrored[col]) {  // the boundary launches already stored the faces
    ctx->mirrored[col] = false;
    return KGS_OK;
  }
  const size_t face = (size_t)3 * ctx->pp;
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaEventRecord(s.ev_bnd, s.stream));
  }
  if (ctx->dist) {
    Slab& s = ctx->slabs[0];
    const int up = (ctx->rank + 1) % ctx->nranks;
    const int dn = (ctx->rank - 1 + ctx->nranks) % ctx->nranks;
    double* p0 = s.plane0[col];
    CK(cudaStreamWaitEvent(s.cstream, s.ev_bnd, 0));
    NK(g_nccl.GroupStart());
    // order matters when up == dn (2 ranks): sends [to dn: plane 0, to up:
    // plane nx-1]; recvs [from up: ghost nx, from dn: ghost -1].
    NK(g_nccl.Send(p0, face, ncclFloat64, dn, ctx->comm, s.cstream));
    NK(g_nccl.Send(p0 + (int64_t)(s.nx - 1) * ctx->ps, face, ncclFloat64, up,
                   ctx->comm, s.cstream));
    NK(g_nccl.Recv(p0 + (int64_t)s.nx * ctx->ps, face, ncclFloat64, up,
                   ctx->comm, s.cstream));
    NK(g_nccl.Recv(p0 - ctx->ps, face, ncclFloat64, dn, ctx->comm, s.cstream));
    NK(g_nccl.GroupEnd());
    CK(cudaEventRecord(s.ev_xch, s.cstream));
    s.xch_pending = true;
    return KGS_OK;
  }
  const int ns = (int)ctx->slabs.size();
  for (int i = 0; i < ns; ++i) {
    Slab& s = ctx->slabs[i];
    Slab& lo = ctx->slabs[(i - 1 + ns) % ns];
    Slab& hi = ctx->slabs[(i + 1) % ns];
    CK(cudaSetDevice(s.dev));
    // own boundary pass done (it read these ghosts' previous contents) and
    // the neighbours' faces written
    CK(cudaStreamWaitEvent(s.cstream, s.ev_bnd, 0));
    CK(cudaStreamWaitEvent(s.cstream, lo.ev_bnd, 0));
    CK(cudaStreamWaitEvent(s.cstream, hi.ev_bnd, 0));
    // pull: ghost -1 <- lo plane nx-1 ; ghost nx <- hi plane 0
    double* g_lo = s.plane0[col] - ctx->ps;
    double* g_hi = s.plane0[col] + (int64_t)s.nx * ctx->ps;
    const double* src_lo = lo.plane0[col] + (int64_t)(lo.nx - 1) * ctx->ps;
    const double* src_hi = hi.plane0[col];
    if (lo.dev == s.dev)
      CK(cudaMemcpyAsync(g_lo, src_lo, face * 8, cudaMemcpyDeviceToDevice, s.cstream));
    else
      CK(cudaMemcpyPeerAsync(g_lo, s.dev, src_lo, lo.dev, face * 8, s.cstream));
    if (hi.dev == s.dev)
      CK(cudaMemcpyAsync(g_hi, src_hi, face * 8, cudaMemcpyDeviceToDevice, s.cstream));
    else
      CK(cudaMemcpyPeerAsync(g_hi, s.dev, src_hi, hi.dev, face * 8, s.cstream));
    CK(cudaEventRecord(s.ev_xch, s.cstream));
    s.xch_pending = true;
  }
  // A face read by a neighbour's pull in exchange k is next overwritten by
  // this slab's boundary pass k+2, which waits for this slab's exchange k+1,
  // which waits (ev_bnd) for the neighbour's boundary pass k+1, which waits
  // for the neighbour's exchange k: ordered.
  return KGS_OK;
}

int sync_all(kgs_ctx* ctx) {
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.stream));
    CK(cudaStreamSynchronize(s.cstream));
  }
  return KGS_OK;
}

// One colour pass over every slab.  With several slabs (or ranks) the
// interior planes [1, nx-1) go first -- they need no ghost data, so they
// overlap the previous pass's halo exchange -- then the stream waits for
// that exchange (ev_xch) and runs the two boundary planes.
//
// Fused halo exchange (ctx->mirror): the boundary launches of slab i also
// store their new faces into the neighbours' ghost planes (peer pointers),
// so no exchange follows.  Before slab i's boundary launches of pass k its
// stream waits for both neighbours' boundary launches of pass k-1 (ev_face):
// that is when they finished writing i's ghosts (RAW) and finished reading
// their own ghosts that i is about to overwrite (WAR); pending copy
// exchanges into either side are waited for as well.
int all_passes(kgs_ctx* ctx, int col, int op1, int op2, bool diag, bool check,
               const Coeffs& c, int step_no) {
  const bool split = needs_exchange(ctx);
  const bool mirror = split && ctx->mirror && ctx->tune_mirror;
  const bool writes = op1 != OP_NONE || op2 != OP_NONE;
  const int64_t k = ctx->pass_no;
  if (split) ctx->pass_no++;
  const int ns = (int)ctx->slabs.size();
  for (int i = 0; i < ns; ++i) {
    Slab& s = ctx->slabs[i];
    cudaError_t e = cudaSetDevice(s.dev);
    if (e != cudaSuccess) return fail(ctx, KGS_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    if (diag) s.npart[col] = 0;
    int r;
    if (!split) {
      r = launch_pass(ctx, s, col, op1, op2, diag, check, c, step_no);
    } else {
      r = KGS_OK;
      if (s.nx > 2) r = launch_pass(ctx, s, col, op1, op2, diag, check, c, step_no, 1, s.nx - 1);
      if (!r && s.xch_pending) {
        CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
        s.xch_pending = false;
      }
      Slab& lo = ctx->slabs[(i - 1 + ns) % ns];
      Slab& hi = ctx->slabs[(i + 1) % ns];
      if (!r && mirror) {
        CK(cudaStreamWaitEvent(s.stream, lo.ev_xch, 0));
        CK(cudaStreamWaitEvent(s.stream, hi.ev_xch, 0));
        if (k > 0) {
          CK(cudaStreamWaitEvent(s.stream, lo.ev_face[(k - 1) & 1], 0));
          CK(cudaStreamWaitEvent(s.stream, hi.ev_face[(k - 1) & 1], 0));
        }
      }
      // our plane 0 is lo's ghost plane lo.nx; our plane nx-1 is hi's ghost -1
      double* mlo = (mirror && writes) ? lo.plane0[col] + (int64_t)lo.nx * ctx->ps : nullptr;
      double* mhi = (mirror && writes) ? hi.plane0[col] - ctx->ps : nullptr;
      if (!r) r = launch_pass(ctx, s, col, op1, op2, diag, check, c, step_no, 0, 1, nullptr,
                              mlo, nullptr);
      if (!r) r = launch_pass(ctx, s, col, op1, op2, diag, check, c, step_no, s.nx - 1, s.nx,
                              nullptr, nullptr, mhi);
      if (!r && mirror) CK(cudaEventRecord(s.ev_face[k & 1], s.stream));
    }
    if (r) return r;
  }
  if (mirror && writes) ctx->mirrored[col] = true;
  return KGS_OK;
}

// Run `launch` bracketed by an event pair on slab 0's stream when timing.
template <class F>
int timed(kgs_ctx* ctx, int64_t pts, F&& launch) {
  ctx->timed_pts = pts;
  if (!ctx->pass_timing) return launch();
  Slab& s0 = ctx->slabs[0];
  if (ctx->pass_ev_used + 2 > ctx->pass_ev.size()) {
    CK(cudaSetDevice(s0.dev));
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ctx->pass_ev.push_back(e);
    }
  }
  cudaEvent_t a = ctx->pass_ev[ctx->pass_ev_used++];
  cudaEvent_t b = ctx->pass_ev[ctx->pass_ev_used++];
  CK(cudaSetDevice(s0.dev));
  CK(cudaEventRecord(a, s0.stream));
  int r = launch();
  if (r) return r;
  CK(cudaSetDevice(s0.dev));
  CK(cudaEventRecord(b, s0.stream));
  return KGS_OK;
}

// all_passes() bracketed by an event pair on slab 0's stream when timing.
int timed_passes(kgs_ctx* ctx, int col, int op1, int op2, bool diag, bool check,
                 const Coeffs& c, int step_no) {
  int64_t pts = 0;
  for (auto& s : ctx->slabs) pts += (int64_t)s.nx * ctx->ny * ctx->nk;
  ctx->timed_pts = pts;
  if (!ctx->pass_timing) return all_passes(ctx, col, op1, op2, diag, check, c, step_no);
  Slab& s0 = ctx->slabs[0];
  if (ctx->pass_ev_used + 2 > ctx->pass_ev.size()) {
    CK(cudaSetDevice(s0.dev));
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ctx->pass_ev.push_back(e);
    }
  }
  cudaEvent_t a = ctx->pass_ev[ctx->pass_ev_used++];
  cudaEvent_t b = ctx->pass_ev[ctx->pass_ev_used++];
  CK(cudaSetDevice(s0.dev));
  CK(cudaEventRecord(a, s0.stream));
  int r = all_passes(ctx, col, op1, op2, diag, check, c, step_no);
  if (r) return r;
  CK(cudaSetDevice(s0.dev));
  CK(cudaEventRecord(b, s0.stream));
  return KGS_OK;
}

int collect_pass_times(kgs_ctx* ctx) {
  for (size_t i = 0; i + 1 < ctx->pass_ev_used; i += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->pass_ev[i], ctx->pass_ev[i + 1]));
    ctx->pass_ms += ms;
    ctx->pass_count++;
  }
  ctx->pass_ev_used = 0;
  return KGS_OK;
}

int finalize_record(kgs_ctx* ctx, int64_t slot, bool both) {
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    finalize_terms<<<1, kThreads, 0, s.stream>>>(
        s.partials[1], s.npart[1], both ? s.partials[0] : nullptr,
        both ? s.npart[0] : 0, s.records + slot * NTERMS);
    ctx->launches++;
    CK(cudaGetLastError());
  }
  return KGS_OK;
}

// Apply a deferred red adjoint so the resident state is the reference's.
int flush_pending(kgs_ctx* ctx) {
  if (!ctx->pending) return KGS_OK;
  ctx->pending = false;
  int r = all_passes(ctx, 1, OP_ADJ, OP_NONE, false, false, ctx->pend_c, 0);
  if (!r) r = exchange(ctx, 1);
  return r;
}

int ensure_records(kgs_ctx* ctx, int64_t n) {
  for (auto& s : ctx->slabs) {
    if (s.rec_cap >= n) continue;
    CK(cudaSetDevice(s.dev));
    if (s.records) CK(cudaFree(s.records));
    s.records = nullptr;
    const int64_t cap = std::max<int64_t>(n, 64);
    CK(cudaMalloc(&s.records, (size_t)cap * NTERMS * sizeof(double)));
    s.rec_cap = cap;
  }
  return KGS_OK;
}

int reset_bad(kgs_ctx* ctx) {
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaMemsetAsync(s.bad, 0xff, sizeof(unsigned long long), s.stream));
  }
  return KGS_OK;
}

int read_bad(kgs_ctx* ctx, unsigned long long* out) {
  *out = ULLONG_MAX;
  for (auto& s : ctx->slabs) {
    unsigned long long v = 0;
    CK(cudaSetDevice(s.dev));
    CK(cudaMemcpyAsync(&v, s.bad, sizeof v, cudaMemcpyDeviceToHost, s.stream));
    CK(cudaStreamSynchronize(s.stream));
    *out = std::min(*out, v);
  }
  return KGS_OK;
}

Coeffs to_coeffs(const kgs_coeffs* c) {
  Coeffs k;
  static_assert(sizeof(Coeffs) == sizeof(kgs_coeffs), "coeff layout");
  std::memcpy(&k, c, sizeof k);
  return k;
}


int alloc_slab(kgs_ctx* ctx, Slab& s) {
  CK(cudaSetDevice(s.dev));
  const size_t colour_bytes = (size_t)(s.nx + 2) * ctx->ps * sizeof(double);
  for (int c = 0; c < 2; ++c) {
    cudaError_t e = cudaMalloc(&s.buf[c], colour_bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, KGS_ENOMEM, "cudaMalloc of %zu bytes failed: %s",
                  colour_bytes, cudaGetErrorString(e));
    }
    CK(cudaMemset(s.buf[c], 0, colour_bytes));
    s.plane0[c] = s.buf[c] + ctx->ps;
    // up to 3 launches (interior + 2 boundary planes) per pass write partials
    CK(cudaMalloc(&s.partials[c], (size_t)4 * ctx->grid_cap * NTERMS * sizeof(double)));
  }
  if (ctx->d == 3) {
    int r = make_tensor_maps(ctx, s);
    if (r) return r;
  }
  CK(cudaMalloc(&s.bad, sizeof(unsigned long long)));
  CK(cudaMemset(s.bad, 0xff, sizeof(unsigned long long)));
  // staging: up to 256 MiB of natural-layout planes of one field
  const size_t nat_plane = (size_t)ctx->ny * ctx->nz * sizeof(double);
  s.stage_planes = (int)std::max<size_t>(1, std::min<size_t>(s.nx, (256u << 20) / nat_plane));
  CK(cudaMalloc(&s.stage, s.stage_planes * nat_plane));
  CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s.cstream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&s.ev_bnd, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_xch, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i)
    CK(cudaEventCreateWithFlags(&s.ev_face[i], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming));
  CK(cudaEventCreate(&s.ev_t0));
  CK(cudaEventCreate(&s.ev_t1));
  return KGS_OK;
}

int init_geometry(kgs_ctx* ctx, int d, int64_t N, double a, double b) {
  if (d < 1 || d > 3) return fail(ctx, KGS_EINVAL, "dimension must be 1, 2 or 3, got %d", d);
  if (!(b > a)) return fail(ctx, KGS_EINVAL, "need b > a, got a=%g, b=%g", a, b);
  if (N < 2) return fail(ctx, KGS_EINVAL, "need N >= 2, got N=%lld", (long long)N);
  if (N % 2)
    return fail(ctx, KGS_EINVAL,
                "checkerboard needs even N for a consistent periodic 2-coloring, got N=%lld",
                (long long)N);
  if (N > (1 << 20)) return fail(ctx, KGS_EINVAL, "N=%lld too large", (long long)N);
  ctx->d = d;
  ctx->N = N;
  ctx->a = a;
  ctx->b = b;
  ctx->h = (b - a) / (double)N;
  ctx->nz = (int)N;
  ctx->nk = (int)(N / 2);
  ctx->ny = (d == 3) ? (int)N : 1;
  ctx->nxg = (d >= 2) ? N : 1;
  ctx->rs = ctx->nk;
  ctx->pp = (int64_t)ctx->ny * ctx->rs;
  ctx->ps = 4 * ctx->pp;
  return KGS_OK;
}

int init_device_props(kgs_ctx* ctx, int dev) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major < 10)
    return fail(ctx, KGS_ECUDA,
                "device %d is sm_%d%d; this library is built for sm_100a (B200)",
                dev, prop.major, prop.minor);
  ctx->nsm = prop.multiProcessorCount;
  ctx->grid_cap = ctx->nsm * 8;
  return KGS_OK;
}

}  // namespace

// =========================================================================
// extern "C" API
// =========================================================================
extern "C" {

int kgs_abi_version(void) { return 100; }

const char* kgs_last_error(kgs_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

int64_t kgs_launch_count(kgs_ctx* ctx) { return ctx ? ctx->launches : 0; }

double kgs_last_step_ms(kgs_ctx* ctx) { return ctx ? ctx->last_ms : 0.0; }

int kgs_create(int d, int64_t N, double a, double b, int nslabs,
               const int* dev_ids, kgs_ctx** out) {
  if (!out) return fail(nullptr, KGS_EINVAL, "out is NULL");
  *out = nullptr;
  kgs_ctx* ctx = new kgs_ctx();
  int r = init_geometry(ctx, d, N, a, b);
  if (!r && nslabs < 1) r = fail(ctx, KGS_EINVAL, "nslabs must be >= 1");
  if (!r && nslabs > 1 && d == 1) r = fail(ctx, KGS_EINVAL, "1-D grids cannot be split into slabs");
  if (!r && ctx->nxg % nslabs) r = fail(ctx, KGS_EINVAL, "N=%lld not divisible by %d slabs", (long long)N, nslabs);
  if (!r && nslabs > 1 && ctx->nxg / nslabs < 2) r = fail(ctx, KGS_EINVAL, "slabs need >= 2 planes");
  if (!r) r = init_device_props(ctx, dev_ids ? dev_ids[0] : 0);
  if (!r) {
    ctx->slabs.resize(nslabs);
    const int per = (int)(ctx->nxg / nslabs);
    for (int i = 0; i < nslabs && !r; ++i) {
      Slab& s = ctx->slabs[i];
      s.dev = dev_ids ? dev_ids[i] : 0;
      s.x0 = (int64_t)i * per;
      s.nx = per;
      r = alloc_slab(ctx, s);
    }
  }
  if (!r) {  // enable peer access between distinct devices (best effort)
    for (auto& s : ctx->slabs)
      for (auto& t : ctx->slabs)
        if (s.dev != t.dev) {
          cudaSetDevice(s.dev);
          if (cudaDeviceEnablePeerAccess(t.dev, 0) != cudaSuccess) cudaGetLastError();
        }
    // fused halo stores need every slab to reach its neighbours' memory
    const int ns = (int)ctx->slabs.size();
    ctx->mirror = ns > 1;
    for (int i = 0; i < ns && ctx->mirror; ++i)
      for (int dj : {-1, 1}) {
        const int a = ctx->slabs[i].dev, b = ctx->slabs[(i + dj + ns) % ns].dev;
        int ok = 1;
        if (a != b && (cudaDeviceCanAccessPeer(&ok, a, b) != cudaSuccess || !ok)) {
          cudaGetLastError();
          ctx->mirror = false;
        }
      }
  }
  if (r) {
    g_last_error = ctx->err;
    kgs_destroy(ctx);
    return r;
  }
  *out = ctx;
  return KGS_OK;
}

int kgs_nccl_unique_id(void* out128) {
  std::string err;
  if (!load_nccl(err)) return fail(nullptr, KGS_ENCCL, "%s", err.c_str());
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, KGS_ENCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  return KGS_OK;
}

int kgs_create_dist(int d, int64_t N, double a, double b, int rank, int nranks,
                    int device, const void* nccl_id, kgs_ctx** out) {
  if (!out) return fail(nullptr, KGS_EINVAL, "out is NULL");
  *out = nullptr;
  kgs_ctx* ctx = new kgs_ctx();
  ctx->dist = true;
  ctx->rank = rank;
  ctx->nranks = nranks;
  int r = init_geometry(ctx, d, N, a, b);
  if (!r && (nranks < 1 || rank < 0 || rank >= nranks)) r = fail(ctx, KGS_EINVAL, "bad rank %d of %d", rank, nranks);
  if (!r && nranks > 1 && d == 1) r = fail(ctx, KGS_EINVAL, "1-D grids cannot be split into slabs");
  if (!r && ctx->nxg % nranks) r = fail(ctx, KGS_EINVAL, "N=%lld not divisible by %d ranks", (long long)N, nranks);
  if (!r && nranks > 1 && ctx->nxg / nranks < 2) r = fail(ctx, KGS_EINVAL, "slabs need >= 2 planes");
  if (!r) r = init_device_props(ctx, device);
  if (!r) {
    ctx->slabs.resize(1);
    Slab& s = ctx->slabs[0];
    s.dev = device;
    s.nx = (int)(ctx->nxg / nranks);
    s.x0 = (int64_t)rank * s.nx;
    r = alloc_slab(ctx, s);
  }
  if (!r && nranks > 1) {
    std::string err;
    if (!nccl_id) r = fail(ctx, KGS_EINVAL, "nccl_id is NULL");
    else if (!load_nccl(err)) r = fail(ctx, KGS_ENCCL, "%s", err.c_str());
    else {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof id);
      cudaSetDevice(device);
      ncclResult_t nr = g_nccl.CommInitRank(&ctx->comm, nranks, id, rank);
      if (nr != ncclSuccess) r = fail(ctx, KGS_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(nr));
    }
  }
  if (r) {
    g_last_error = ctx->err;
    kgs_destroy(ctx);
    return r;
  }
  *out = ctx;
  return KGS_OK;
}

int kgs_destroy(kgs_ctx* ctx) {
  if (!ctx) return KGS_OK;
  if (ctx->comm && g_nccl.ok) g_nccl.CommDestroy(ctx->comm);
  for (auto e : ctx->pass_ev) cudaEventDestroy(e);
  for (auto& s : ctx->slabs) {
    cudaSetDevice(s.dev);
    if (s.stream) cudaStreamSynchronize(s.stream);
    for (int c = 0; c < 2; ++c) {
      if (s.buf[c]) cudaFree(s.buf[c]);
      if (s.partials[c]) cudaFree(s.partials[c]);
    }
    if (s.records) cudaFree(s.records);
    if (s.bad) cudaFree(s.bad);
    if (s.stage) cudaFree(s.stage);
    for (int c = 0; c < 2; ++c)
      if (s.alt[c]) cudaFree(s.alt[c]);
    if (s.ev_done) cudaEventDestroy(s.ev_done);
    if (s.ev_t0) cudaEventDestroy(s.ev_t0);
    if (s.ev_t1) cudaEventDestroy(s.ev_t1);
    if (s.cstream) cudaStreamSynchronize(s.cstream);
    if (s.ev_bnd) cudaEventDestroy(s.ev_bnd);
    if (s.ev_xch) cudaEventDestroy(s.ev_xch);
    for (int i = 0; i < 2; ++i)
      if (s.ev_face[i]) cudaEventDestroy(s.ev_face[i]);
    if (s.dstream) cudaStreamSynchronize(s.dstream);
    for (auto e : s.pipe_ev) cudaEventDestroy(e);
    if (s.dstream) cudaStreamDestroy(s.dstream);
    if (s.pipe_up) cudaFree(s.pipe_up);
    if (s.pipe_dn) cudaFree(s.pipe_dn);
    if (s.pipe_part) cudaFree(s.pipe_part);
    if (s.cstream) cudaStreamDestroy(s.cstream);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  delete ctx;
  return KGS_OK;
}

int kgs_local_range(kgs_ctx* ctx, int64_t* x0, int64_t* nx, int64_t* points) {
  if (!ctx) return fail(nullptr, KGS_EINVAL, "ctx is NULL");
  int64_t lo = ctx->slabs.front().x0, n = 0;
  for (auto& s : ctx->slabs) n += s.nx;
  if (x0) *x0 = lo;
  if (nx) *nx = n;
  if (points) *points = n * (int64_t)ctx->ny * ctx->nz;
  return KGS_OK;
}

}  // extern "C"

namespace {

// Move planes [xg0, xg0 + n) (global plane indices inside this context) of
// field `fi` between a host array in natural layout (`host` = plane xg0) and
// the colour-split device planes, through each slab's staging buffer.
int transfer_planes(kgs_ctx* ctx, int fi, int64_t xg0, int64_t n, double* host, bool to_device) {
  const int64_t nat_plane = (int64_t)ctx->ny * ctx->nz;
  for (auto& s : ctx->slabs) {
    const int64_t lo = std::max<int64_t>(xg0, s.x0), hi = std::min<int64_t>(xg0 + n, s.x0 + s.nx);
    if (lo >= hi) continue;
    CK(cudaSetDevice(s.dev));
    for (int64_t xg = lo; xg < hi; xg += s.stage_planes) {
      const int nxc = (int)std::min<int64_t>(s.stage_planes, hi - xg);
      const int xs = (int)(xg - s.x0);
      const int64_t cnt = (int64_t)nxc * ctx->ny * ctx->nk;
      const int blocks = (int)std::min<int64_t>((cnt + 255) / 256, (int64_t)ctx->nsm * 16);
      PassGeom g = make_geom(ctx, s, 1, 0, s.nx);   // own = red, oth = black
      g.own += fi * ctx->pp;
      g.oth += fi * ctx->pp;
      double* h = host + (xg - xg0) * nat_plane;
      const size_t bytes = (size_t)nxc * nat_plane * 8;
      if (to_device) {
        CK(cudaMemcpyAsync(s.stage, h, bytes, cudaMemcpyHostToDevice, s.stream));
        split_field<<<blocks, 256, 0, s.stream>>>(s.stage, g, nxc, xs);
      } else {
        merge_field<<<blocks, 256, 0, s.stream>>>(s.stage, g, nxc, xs);
      }
      ctx->launches++;
      CK(cudaGetLastError());
      if (!to_device) CK(cudaMemcpyAsync(h, s.stage, bytes, cudaMemcpyDeviceToHost, s.stream));
    }
    CK(cudaStreamSynchronize(s.stream));
  }
  return KGS_OK;
}

// ---- pipelined host integration (kgs_integrate_host) ---------------------
// Upload, the colour passes of a whole integrate() call and the download
// overlap.  Chunks of C planes arrive in folded order (block 0, the last
// block, block 1, the one before, ...), so the arrived region is a periodic
// interval around plane 0 that grows on alternating sides.  Every pass reads
// the other colour at x-1..x+1 and overwrites what its predecessor read, so
// pass j may cover its predecessor's done region shrunk by one plane on each
// side (RAW and WAR at once); the whole ring once the predecessor has it.
// All passes therefore advance as a wavefront behind the upload, on the
// compute stream in dependency order, and a C-plane block is downloaded
// (merge kernel + D2H on a third stream) as soon as the last pass covered it:
// H2D, compute and D2H proceed together (PCIe is full duplex).  The initial
// state is also copied device-side (the second buffer set) so a non-finite
// step can be replayed exactly.  Records get their own partial regions (the
// DIAG passes of different steps are in flight together).
int ensure_alt(kgs_ctx* ctx) {
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    const size_t colour_bytes = (size_t)(s.nx + 2) * ctx->ps * sizeof(double);
    for (int c = 0; c < 2; ++c) {
      if (s.alt[c]) continue;
      if (cudaMalloc(&s.alt[c], colour_bytes) != cudaSuccess) {
        cudaGetLastError();
        s.alt[c] = nullptr;
        return KGS_ENOMEM;
      }
      s.alt0[c] = s.alt[c] + ctx->ps;
    }
  }
  return KGS_OK;
}

struct PipePass {
  int col, op1, op2;
  bool diag, check;
  int step_no;
  int rec;      // record of its DIAG partials (-1: none)
  int shrink;   // planes given up on each side relative to the predecessor
};

constexpr int kPipeFallback = 1;   // not eligible / no memory: use the plain path

// The pipeline as a list of events, in the order they are issued on the
// compute stream: ARRIVE (wait for chunk m = planes [a, b)), PASS (pass j
// over planes [a, b)), FINAL (planes [a, b) are final: copy them back).
// Pure host logic (kgs_pipeline_plan exports it for the CPU tests).
enum PipeKind : int { PIPE_ARRIVE = 0, PIPE_PASS = 1, PIPE_FINAL = 2 };
struct PipeEvent {
  int kind, pass;
  int64_t a, b;
};

std::vector<PipeEvent> pipeline_plan(int64_t N, int64_t C, const std::vector<int>& shrink) {
  std::vector<PipeEvent> ev;
  const int64_t nb = (N + C - 1) / C;
  const int J = (int)shrink.size();
  std::vector<int64_t> lo(J, 0), hi(J, 0);   // done regions, unwrapped: empty or lo < hi
  std::vector<char> full(J, 0), dl(nb, 0);
  auto pass = [&](int j, int64_t a, int64_t b) {
    if (b > a) ev.push_back({PIPE_PASS, j, a, b});
  };
  auto pass_u = [&](int j, int64_t u0, int64_t u1) {   // unwrapped range, u1 - u0 <= N
    if (u1 <= u0) return;
    while (u0 < 0) { u0 += N; u1 += N; }
    while (u0 >= N) { u0 -= N; u1 -= N; }
    if (u1 <= N) pass(j, u0, u1);
    else { pass(j, u0, N); pass(j, 0, u1 - N); }
  };
  int64_t alo = 0, ahi = 0;
  for (int64_t m = 0; m < nb; ++m) {
    const int64_t blk = (m % 2 == 0) ? m / 2 : nb - 1 - m / 2;   // folded order
    const int64_t x0 = blk * C, x1 = std::min(N, x0 + C);
    ev.push_back({PIPE_ARRIVE, (int)m, x0, x1});
    if (m % 2 == 0) ahi = x1; else alo = x0 - N;
    int64_t plo = alo, phi = ahi;
    bool pfull = m == nb - 1;
    for (int j = 0; j < J; ++j) {
      if (!full[j]) {
        if (pfull) {   // the rest of the ring; the region need not contain plane 0
          if (lo[j] == hi[j]) pass(j, 0, N);
          else pass_u(j, hi[j], lo[j] + N);
          full[j] = 1;
        } else {
          const int64_t nlo = plo + shrink[j], nhi = phi - shrink[j];
          if (nhi > nlo) {
            if (lo[j] == hi[j]) pass_u(j, nlo, nhi);
            else { pass_u(j, nlo, lo[j]); pass_u(j, hi[j], nhi); }
            lo[j] = nlo;
            hi[j] = nhi;
          }
        }
      }
      pfull = full[j];
      plo = lo[j];
      phi = hi[j];
    }
    // blocks wholly inside the last pass's done region (which need not
    // contain plane 0 yet) are final
    const int64_t L = lo[J - 1], H = hi[J - 1];
    for (int64_t k = 0; k < nb; ++k) {
      if (dl[k]) continue;
      const int64_t b0 = k * C, b1 = std::min(N, b0 + C);
      if (full[J - 1] || (L < H && ((b0 >= L && b1 <= H) || (b0 - N >= L && b1 - N <= H)))) {
        dl[k] = 1;
        ev.push_back({PIPE_FINAL, (int)k, b0, b1});
      }
    }
  }
  return ev;
}

std::vector<int> pipeline_shrinks(int64_t nsteps) {
  // initial energy (black self, red edges + self), head, then K3/K4 per step
  std::vector<int> sh = {0, 1, 0};
  for (int64_t i = 0; i < 2 * nsteps; ++i) sh.push_back(1);
  return sh;
}

int integrate_pipelined(kgs_ctx* ctx, double* const host[4], const Coeffs& c, int64_t nsteps,
                        int64_t step_offset, int64_t record_stride, int64_t nrec,
                        unsigned long long* bad_out) {
  if (!ctx->tune_pipe || ctx->slabs.size() != 1 || ctx->dist || ctx->d != 3)
    return kPipeFallback;
  Slab& s = ctx->slabs[0];
  const int64_t N = s.nx;
  const int64_t C = std::max<int64_t>(1, ctx->tune_pipe_chunk);
  const int64_t nb = (N + C - 1) / C;
  if (nb < 4) return kPipeFallback;
  const int64_t nat_plane = (int64_t)ctx->ny * ctx->nz;
  CK(cudaSetDevice(s.dev));
  if (ensure_alt(ctx)) return kPipeFallback;
  const int64_t stage = 4 * C * nat_plane;
  if (s.pipe_stage < stage) {
    if (s.pipe_up) CK(cudaFree(s.pipe_up));
    if (s.pipe_dn) CK(cudaFree(s.pipe_dn));
    s.pipe_up = s.pipe_dn = nullptr;
    s.pipe_stage = 0;
    if (cudaMalloc(&s.pipe_up, stage * 8) != cudaSuccess ||
        cudaMalloc(&s.pipe_dn, stage * 8) != cudaSuccess) {
      cudaGetLastError();
      if (s.pipe_up) cudaFree(s.pipe_up);
      s.pipe_up = nullptr;
      return kPipeFallback;
    }
    s.pipe_stage = stage;
  }
  const int64_t maxl = nb + 4;                                 // launches per pass
  const int64_t region = maxl * ctx->grid_cap * NTERMS;        // doubles per (record, colour)
  const int64_t need = (nrec + 1) * 2 * region;
  if (s.pipe_part_cap < need) {
    if (need > (int64_t)1 << 27) return kPipeFallback;         // > 1 GiB of partials
    if (s.pipe_part) CK(cudaFree(s.pipe_part));
    s.pipe_part = nullptr;
    s.pipe_part_cap = 0;
    if (cudaMalloc(&s.pipe_part, need * 8) != cudaSuccess) {
      cudaGetLastError();
      return kPipeFallback;
    }
    s.pipe_part_cap = need;
  }
  if (!s.dstream) CK(cudaStreamCreateWithFlags(&s.dstream, cudaStreamNonBlocking));
  while ((int64_t)s.pipe_ev.size() < 2 * nb) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s.pipe_ev.push_back(e);
  }
  int r = ensure_records(ctx, nrec + 1);
  if (!r) r = reset_bad(ctx);
  if (r) return r;
  ctx->pending = false;   // the whole state is replaced

  // the passes of the call: initial energy (black self, red edges + self),
  // head, then K3(n), K4(n) per step (K4 of the last step = the tail)
  std::vector<PipePass> passes;
  passes.push_back({0, OP_NONE, OP_NONE, true, false, 0, 0, 0});
  passes.push_back({1, OP_NONE, OP_NONE, true, false, 0, 0, 1});
  passes.push_back({1, OP_BASE, OP_NONE, false, false, 0, -1, 0});
  int64_t slot = 0;
  for (int64_t i = 1; i <= nsteps; ++i) {
    const int64_t n = step_offset + i;
    const bool rec = record_stride > 0 && n % record_stride == 0;
    const int rid = rec ? (int)(1 + slot++) : -1;
    passes.push_back({0, OP_BASE, OP_ADJ, rec, true, (int)n, rid, 1});
    passes.push_back({1, OP_ADJ, i < nsteps ? OP_BASE : OP_NONE, rec, true, (int)n, rid, 1});
  }
  const int J = (int)passes.size();
  std::vector<int64_t> roff((size_t)(nrec + 1) * 2, 0);
  std::vector<int> shrink(J);
  for (int j = 0; j < J; ++j) shrink[j] = passes[j].shrink;
  const std::vector<PipeEvent> plan = pipeline_plan(N, C, shrink);

  auto launch_range = [&](const PipePass& P, int64_t xa, int64_t xb) -> int {
    if (xb <= xa) return KGS_OK;
    double* save = s.partials[P.col];
    const int64_t ri = P.diag ? (int64_t)P.rec * 2 + P.col : 0;
    if (P.diag) {
      s.partials[P.col] = s.pipe_part + ri * region;
      s.npart[P.col] = (int)roff[ri];
    }
    int rr = launch_pass(ctx, s, P.col, P.op1, P.op2, P.diag, P.check, c, P.step_no, (int)xa,
                         (int)xb);
    if (P.diag) {
      roff[ri] = s.npart[P.col];
      s.partials[P.col] = save;
    }
    return rr;
  };

  CK(cudaEventRecord(s.ev_t0, s.cstream));
  // uploads (folded block order) on the comm stream: H2D, split, backup copy
  for (const PipeEvent& e : plan) {
    if (e.kind != PIPE_ARRIVE) continue;
    const int64_t m = e.pass, x0 = e.a, x1 = e.b, nxc = x1 - x0;
    for (int f = 0; f < 4; ++f)
      CK(cudaMemcpyAsync(s.pipe_up + f * C * nat_plane, host[f] + x0 * nat_plane,
                         (size_t)nxc * nat_plane * 8, cudaMemcpyHostToDevice, s.cstream));
    const int64_t cnt = nxc * ctx->ny * ctx->nk;
    const int blocks = (int)std::min<int64_t>((cnt + 255) / 256, (int64_t)ctx->nsm * 16);
    for (int f = 0; f < 4; ++f) {
      PassGeom g = make_geom(ctx, s, 1, 0, s.nx);   // own = red, oth = black
      g.own += f * ctx->pp;
      g.oth += f * ctx->pp;
      split_field<<<blocks, 256, 0, s.cstream>>>(s.pipe_up + f * C * nat_plane, g, (int)nxc,
                                                  (int)x0);
      ctx->launches++;
    }
    CK(cudaGetLastError());
    for (int cc = 0; cc < 2; ++cc)
      CK(cudaMemcpyAsync(s.alt0[cc] + x0 * ctx->ps, s.plane0[cc] + x0 * ctx->ps,
                         (size_t)nxc * ctx->ps * 8, cudaMemcpyDeviceToDevice, s.cstream));
    CK(cudaEventRecord(s.pipe_ev[m], s.cstream));
  }

  // the wavefront on the compute stream; downloads behind it
  int64_t ndl = 0;
  for (const PipeEvent& e : plan) {
    if (r) break;
    if (e.kind == PIPE_ARRIVE) {
      CK(cudaStreamWaitEvent(s.stream, s.pipe_ev[e.pass], 0));
    } else if (e.kind == PIPE_PASS) {
      r = launch_range(passes[e.pass], e.a, e.b);
    } else {
      const int64_t k = e.pass, b0 = e.a, nxc = e.b - e.a;
      ++ndl;
      cudaEvent_t ev = s.pipe_ev[nb + k];
      CK(cudaEventRecord(ev, s.stream));
      CK(cudaStreamWaitEvent(s.dstream, ev, 0));
      const int64_t cnt = nxc * ctx->ny * ctx->nk;
      const int blocks = (int)std::min<int64_t>((cnt + 255) / 256, (int64_t)ctx->nsm * 16);
      for (int f = 0; f < 4; ++f) {
        PassGeom g = make_geom(ctx, s, 1, 0, s.nx);
        g.own += f * ctx->pp;
        g.oth += f * ctx->pp;
        merge_field<<<blocks, 256, 0, s.dstream>>>(s.pipe_dn + f * C * nat_plane, g, (int)nxc,
                                                    (int)b0);
        ctx->launches++;
        CK(cudaMemcpyAsync(host[f] + b0 * nat_plane, s.pipe_dn + f * C * nat_plane,
                           (size_t)nxc * nat_plane * 8, cudaMemcpyDeviceToHost, s.dstream));
      }
      CK(cudaGetLastError());
    }
  }
  if (r) return r;
  if (ndl != nb) return fail(ctx, KGS_ECUDA, "pipeline copied back %lld of %lld blocks",
                             (long long)ndl, (long long)nb);
  for (int64_t q = 0; q <= nrec; ++q) {
    finalize_terms<<<1, kThreads, 0, s.stream>>>(
        s.pipe_part + (q * 2 + 1) * region, (int)roff[q * 2 + 1], s.pipe_part + (q * 2) * region,
        (int)roff[q * 2], s.records + q * NTERMS);
    ctx->launches++;
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(s.ev_done, s.dstream));
  CK(cudaStreamWaitEvent(s.stream, s.ev_done, 0));
  CK(cudaEventRecord(s.ev_t1, s.stream));
  r = sync_all(ctx);
  if (!r) CK(cudaStreamSynchronize(s.dstream));
  if (r) return r;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, s.ev_t0, s.ev_t1));
  ctx->last_ms = ms;
  return read_bad(ctx, bad_out);
}

int check_range(kgs_ctx* ctx, int field, int64_t xg0, int64_t n, const void* p) {
  if (!ctx || !p) return fail(ctx, KGS_EINVAL, "NULL argument");
  if (field < 0 || field > 3) return fail(ctx, KGS_EINVAL, "field must be 0..3 (P, Q, U, V)");
  int64_t lo = ctx->slabs.front().x0, cnt = 0;
  for (auto& s : ctx->slabs) cnt += s.nx;
  if (n < 0 || xg0 < lo || xg0 + n > lo + cnt)
    return fail(ctx, KGS_EINVAL, "planes [%lld, %lld) outside this context's [%lld, %lld)",
                (long long)xg0, (long long)(xg0 + n), (long long)lo, (long long)(lo + cnt));
  return KGS_OK;
}

}  // namespace

extern "C" {

int kgs_upload(kgs_ctx* ctx, const double* P, const double* Q, const double* U,
               const double* V) {
  if (!ctx || !P || !Q || !U || !V) return fail(ctx, KGS_EINVAL, "NULL argument");
  ctx->pending = false;  // the whole state is replaced
  const double* f[4] = {P, Q, U, V};
  int64_t x0, nx;
  kgs_local_range(ctx, &x0, &nx, nullptr);
  for (int fi = 0; fi < 4; ++fi) {
    int r = transfer_planes(ctx, fi, x0, nx, const_cast<double*>(f[fi]), true);
    if (r) return r;
  }
  ctx->mirrored[0] = ctx->mirrored[1] = false;  // planes written without mirroring
  int r = exchange(ctx, 0);
  if (!r) r = exchange(ctx, 1);
  if (!r) r = sync_all(ctx);
  return r;
}

int kgs_download(kgs_ctx* ctx, double* P, double* Q, double* U, double* V) {
  if (!ctx || !P || !Q || !U || !V) return fail(ctx, KGS_EINVAL, "NULL argument");
  if (int r0 = flush_pending(ctx)) return r0;
  double* f[4] = {P, Q, U, V};
  int64_t x0, nx;
  kgs_local_range(ctx, &x0, &nx, nullptr);
  for (int fi = 0; fi < 4; ++fi) {
    int r = transfer_planes(ctx, fi, x0, nx, f[fi], false);
    if (r) return r;
  }
  return KGS_OK;
}

int kgs_upload_planes(kgs_ctx* ctx, int field, int64_t x_begin, int64_t nplanes,
                      const double* src) {
  int r = check_range(ctx, field, x_begin, nplanes, src);
  if (!r) r = flush_pending(ctx);
  if (!r) r = transfer_planes(ctx, field, x_begin, nplanes, const_cast<double*>(src), true);
  ctx->mirrored[0] = ctx->mirrored[1] = false;  // planes written without mirroring
  if (!r && field < 3) r = exchange(ctx, 0);   // refresh faces (P, Q, U are halo fields)
  if (!r && field < 3) r = exchange(ctx, 1);
  if (!r) r = sync_all(ctx);
  return r;
}

int kgs_download_planes(kgs_ctx* ctx, int field, int64_t x_begin, int64_t nplanes,
                        double* dst) {
  int r = check_range(ctx, field, x_begin, nplanes, dst);
  if (!r) r = flush_pending(ctx);
  if (!r) r = transfer_planes(ctx, field, x_begin, nplanes, dst, false);
  return r;
}

int kgs_sweep(kgs_ctx* ctx, int colour, int kind, const kgs_coeffs* c) {
  if (!ctx || !c) return fail(ctx, KGS_EINVAL, "NULL argument");
  if (colour != 0 && colour != 1) return fail(ctx, KGS_EINVAL, "colour must be 0 or 1");
  if (kind != 0 && kind != 1) return fail(ctx, KGS_EINVAL, "kind must be 0 (base) or 1 (adjoint)");
  const Coeffs k = to_coeffs(c);
  int r = flush_pending(ctx);
  if (!r) r = all_passes(ctx, colour, kind == 0 ? OP_BASE : OP_ADJ, OP_NONE, false, false, k, 0);
  if (!r) r = exchange(ctx, colour);
  if (!r) r = sync_all(ctx);
  return r;
}

int kgs_step_dpavf2(kgs_ctx* ctx, const kgs_coeffs* half, int64_t nsteps,
                    int64_t step_offset, int64_t record_stride,
                    double* terms_out, int64_t* first_bad_step, int flags) {
  if (!ctx || !half) return fail(ctx, KGS_EINVAL, "NULL argument");
  if (nsteps < 0 || record_stride < 0 || step_offset < 0)
    return fail(ctx, KGS_EINVAL, "negative nsteps/step_offset/record_stride");
  if (first_bad_step) *first_bad_step = 0;
  if (nsteps == 0) return KGS_OK;
  if (nsteps + step_offset > INT_MAX) return fail(ctx, KGS_EINVAL, "step numbers too large");
  const int64_t nrec = record_stride > 0
      ? (step_offset + nsteps) / record_stride - step_offset / record_stride : 0;
  if (nrec > 0 && !terms_out) return fail(ctx, KGS_EINVAL, "terms_out is NULL");
  const Coeffs c = to_coeffs(half);
  int r = ensure_records(ctx, nrec);
  if (!r) r = reset_bad(ctx);
  if (r) return r;
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaEventRecord(s.ev_t0, s.stream));
  }
  const int64_t last = step_offset + nsteps;
  const bool defer = (flags & KGS_STEP_DEFER_TAIL) &&
                     !(record_stride > 0 && last % record_stride == 0);
  const bool resident = resident_eligible(ctx);
  // head: base red(first step) -- fused with a deferred red adjoint of the
  // previous call when its coefficients are the same (bitwise neutral)
  const bool head_fused = ctx->pending && std::memcmp(&ctx->pend_c, &c, sizeof c) == 0;
  if (head_fused) {
    ctx->pending = false;
    if (!resident) r = all_passes(ctx, 1, OP_ADJ, OP_BASE, false, false, c, 0);
  } else {
    r = flush_pending(ctx);
    if (!r && !resident) r = all_passes(ctx, 1, OP_BASE, OP_NONE, false, false, c, 0);
  }
  if (!r && resident) {
    // the whole call in one launch (state in shared memory)
    r = launch_resident(ctx, c, nsteps, step_offset, record_stride, head_fused, defer);
    if (!r && defer) {
      ctx->pending = true;
      ctx->pend_c = c;
    }
    nsteps = 0;   // skip the per-step loop below
  }
  if (!r && !resident) r = exchange(ctx, 1);
  int64_t slot = 0;
  const bool fused = fused_ready(ctx);
  int64_t all_pts = 0;
  for (auto& s : ctx->slabs) all_pts += (int64_t)s.nx * ctx->ny * ctx->nk * 2;
  for (int64_t i = 1; i <= nsteps && !r; ++i) {
    const int64_t n = step_offset + i;
    const bool rec = record_stride > 0 && n % record_stride == 0;
    if (fused && !(i == nsteps && defer)) {
      // one fused march: K3(n) and K4(n) (the tail adjoint on the last step)
      r = timed(ctx, all_pts, [&] { return step_fused(ctx, rec, i == nsteps, c, (int)n); });
      if (!r && rec) r = finalize_record(ctx, slot++, false);
      continue;
    }
    // K3: black base(n) + adjoint(n)
    r = timed_passes(ctx, 0, OP_BASE, OP_ADJ, rec, true, c, (int)n);
    if (!r) r = exchange(ctx, 0);
    // K4: red adjoint(n) + base(n+1), or the tail: red adjoint(last)
    if (!r && i < nsteps) r = timed_passes(ctx, 1, OP_ADJ, OP_BASE, rec, true, c, (int)n);
    else if (!r && defer) {  // leave the red adjoint of the last step pending
      ctx->pending = true;
      ctx->pend_c = c;
      break;
    } else if (!r) r = all_passes(ctx, 1, OP_ADJ, OP_NONE, rec, true, c, (int)n);
    if (!r) r = exchange(ctx, 1);
    if (!r && rec) r = finalize_record(ctx, slot++, true);
  }
  if (r) return r;
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    // the step ends when the last halo exchange has landed
    if (s.xch_pending) CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
    CK(cudaEventRecord(s.ev_t1, s.stream));
  }
  r = sync_all(ctx);
  if (r) return r;
  double ms = 0.0;
  for (auto& s : ctx->slabs) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, s.ev_t0, s.ev_t1));
    ms = std::max(ms, (double)t);
  }
  ctx->last_ms = ms;
  r = collect_pass_times(ctx);
  if (r) return r;
  if (nrec > 0) {
    std::vector<double> tmp((size_t)nrec * NTERMS);
    std::fill(terms_out, terms_out + nrec * NTERMS, 0.0);
    for (auto& s : ctx->slabs) {  // slab order: deterministic host sum
      CK(cudaSetDevice(s.dev));
      CK(cudaMemcpy(tmp.data(), s.records, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (size_t q = 0; q < tmp.size(); ++q) terms_out[q] += tmp[q];
    }
  }
  unsigned long long bad = 0;
  r = read_bad(ctx, &bad);
  if (r) return r;
  if (bad != ULLONG_MAX) {
    if (first_bad_step) *first_bad_step = (int64_t)bad;
    return fail(ctx, KGS_ENONFINITE, "non-finite field values detected after step %llu", bad);
  }
  return KGS_OK;
}

int kgs_energy_terms(kgs_ctx* ctx, double* terms_out) {
  if (!ctx || !terms_out) return fail(ctx, KGS_EINVAL, "NULL argument");
  Coeffs dummy{};
  int r = flush_pending(ctx);
  if (!r) r = ensure_records(ctx, 1);
  // red: edges + red self terms; black: black self terms
  if (!r) r = all_passes(ctx, 1, OP_NONE, OP_NONE, true, false, dummy, 0);
  if (!r) r = all_passes(ctx, 0, OP_NONE, OP_NONE, true, false, dummy, 0);
  if (!r) r = finalize_record(ctx, 0, true);
  if (!r) r = sync_all(ctx);
  if (r) return r;
  std::fill(terms_out, terms_out + NTERMS, 0.0);
  for (auto& s : ctx->slabs) {
    double tmp[NTERMS];
    CK(cudaSetDevice(s.dev));
    CK(cudaMemcpy(tmp, s.records, sizeof tmp, cudaMemcpyDeviceToHost));
    for (int q = 0; q < NTERMS; ++q) terms_out[q] += tmp[q];
  }
  return KGS_OK;
}

int64_t kgs_pipeline_plan(int64_t N, int64_t C, int64_t nsteps, int64_t* out, int64_t cap) {
  if (N < 1 || C < 1 || nsteps < 0) return -1;
  const std::vector<PipeEvent> plan = pipeline_plan(N, C, pipeline_shrinks(nsteps));
  const int64_t n = (int64_t)plan.size();
  for (int64_t i = 0; i < std::min(n, cap); ++i) {
    out[4 * i] = plan[i].kind;
    out[4 * i + 1] = plan[i].pass;
    out[4 * i + 2] = plan[i].a;
    out[4 * i + 3] = plan[i].b;
  }
  return n;
}

int kgs_integrate_host(kgs_ctx* ctx, double* P, double* Q, double* U, double* V,
                       const kgs_coeffs* half, int64_t nsteps, int64_t step_offset,
                       int64_t record_stride, double* terms0, double* terms_out,
                       int64_t* first_bad_step, int flags) {
  (void)flags;
  if (!ctx || !P || !Q || !U || !V || !half || !terms0)
    return fail(ctx, KGS_EINVAL, "NULL argument");
  if (nsteps < 0 || record_stride < 0 || step_offset < 0)
    return fail(ctx, KGS_EINVAL, "negative nsteps/step_offset/record_stride");
  if (nsteps + step_offset > INT_MAX) return fail(ctx, KGS_EINVAL, "step numbers too large");
  if (first_bad_step) *first_bad_step = 0;
  const int64_t nrec = record_stride > 0
      ? (step_offset + nsteps) / record_stride - step_offset / record_stride : 0;
  if (nrec > 0 && !terms_out) return fail(ctx, KGS_EINVAL, "terms_out is NULL");
  double* host[4] = {P, Q, U, V};
  const Coeffs c = to_coeffs(half);
  unsigned long long bad = ULLONG_MAX;
  int r = nsteps > 0 ? integrate_pipelined(ctx, host, c, nsteps, step_offset, record_stride,
                                          nrec, &bad)
                     : kPipeFallback;
  if (r == kPipeFallback) {
    // plain path: upload, initial energy, steps, download
    r = kgs_upload(ctx, P, Q, U, V);
    if (!r) r = kgs_energy_terms(ctx, terms0);
    if (r) return r;
    int64_t fb = 0;
    r = kgs_step_dpavf2(ctx, half, nsteps, step_offset, record_stride, terms_out, &fb, 0);
    if (r && r != KGS_ENONFINITE) return r;
    if (r == KGS_ENONFINITE) {   // replay from the (untouched) host state to the bad step
      int r2 = kgs_upload(ctx, P, Q, U, V);
      int64_t fb2 = 0;
      if (!r2 && fb > step_offset)
        r2 = kgs_step_dpavf2(ctx, half, fb - step_offset, step_offset, 0, nullptr, &fb2, 0);
      if (r2 && r2 != KGS_ENONFINITE) return r2;
      if (first_bad_step) *first_bad_step = fb;
      int r3 = kgs_download(ctx, P, Q, U, V);
      if (r3) return r3;
      return fail(ctx, KGS_ENONFINITE, "non-finite field values detected after step %lld",
                  (long long)fb);
    }
    return kgs_download(ctx, P, Q, U, V);
  }
  if (r) return r;
  Slab& s = ctx->slabs[0];
  std::vector<double> rec((size_t)(nrec + 1) * NTERMS);
  CK(cudaMemcpy(rec.data(), s.records, rec.size() * sizeof(double), cudaMemcpyDeviceToHost));
  std::copy(rec.begin(), rec.begin() + NTERMS, terms0);
  if (nrec > 0) std::copy(rec.begin() + NTERMS, rec.end(), terms_out);
  if (bad != ULLONG_MAX) {
    // restore the initial state (device copy) and replay exactly to the bad step
    for (int cc = 0; cc < 2; ++cc)
      CK(cudaMemcpy(s.buf[cc], s.alt[cc], (size_t)(s.nx + 2) * ctx->ps * 8,
                    cudaMemcpyDeviceToDevice));
    int64_t fb2 = 0;
    r = KGS_OK;
    if ((int64_t)bad > step_offset)
      r = kgs_step_dpavf2(ctx, half, (int64_t)bad - step_offset, step_offset, 0, nullptr, &fb2,
                          0);
    if (r && r != KGS_ENONFINITE) return r;
    r = kgs_download(ctx, P, Q, U, V);
    if (r) return r;
    if (first_bad_step) *first_bad_step = (int64_t)bad;
    return fail(ctx, KGS_ENONFINITE, "non-finite field values detected after step %llu", bad);
  }
  return KGS_OK;
}

int kgs_energy_mass(kgs_ctx* ctx, double kappa1, double kappa2, double mu,
                    double gamma, double* E, double* mass) {
  double t[NTERMS];
  int r = kgs_energy_terms(ctx, t);
  if (r) return r;
  const double h = ctx->h, h2 = h * h;
  double hd = 1.0;
  for (int i = 0; i < ctx->d; ++i) hd *= h;
  const double quad = kappa1 * (t[0] / h2) + kappa1 * (t[1] / h2) +
                      kappa2 * (t[2] / h2) + t[3] + mu * mu * t[4];
  if (E) *E = hd * (0.5 * quad - gamma * t[5]);
  if (mass) *mass = hd * (t[6] + t[7]);
  return KGS_OK;
}

int kgs_all_finite(kgs_ctx* ctx, int* ok) {
  if (!ctx || !ok) return fail(ctx, KGS_EINVAL, "NULL argument");
  Coeffs dummy{};
  int r = flush_pending(ctx);
  if (!r) r = reset_bad(ctx);
  if (!r) r = all_passes(ctx, 1, OP_NONE, OP_NONE, false, true, dummy, 1);
  if (!r) r = all_passes(ctx, 0, OP_NONE, OP_NONE, false, true, dummy, 1);
  if (!r) r = sync_all(ctx);
  if (r) return r;
  unsigned long long bad = 0;
  r = read_bad(ctx, &bad);
  if (r) return r;
  *ok = (bad == ULLONG_MAX) ? 1 : 0;
  return KGS_OK;
}

int kgs_host_alloc(int64_t bytes, void** out) {
  kgs_ctx* ctx = nullptr;
  if (!out || bytes < 0) return fail(nullptr, KGS_EINVAL, "bad arguments");
  *out = nullptr;
  CK(cudaHostAlloc(out, (size_t)std::max<int64_t>(bytes, 8), cudaHostAllocPortable));
  return KGS_OK;
}

int kgs_host_free(void* p) {
  kgs_ctx* ctx = nullptr;
  if (p) CK(cudaFreeHost(p));
  return KGS_OK;
}

int kgs_set_tuning(kgs_ctx* ctx, int rows_per_tile, int band_rows, int blocks_per_sm,
                   int march_planes, int march_variant) {
  if (!ctx) return fail(nullptr, KGS_EINVAL, "ctx is NULL");
  if (rows_per_tile < 1 || rows_per_tile > kThreads || (rows_per_tile & (rows_per_tile - 1)))
    return fail(ctx, KGS_EINVAL, "rows_per_tile must be a power of two in [1, 256]");
  ctx->tune_ty = rows_per_tile;
  ctx->tune_band_rows = band_rows;
  ctx->tune_occ = blocks_per_sm;
  ctx->tune_xc = march_planes;
  if (march_variant >= 0) ctx->tune_variant = march_variant;
  return KGS_OK;
}

int kgs_debug_pass(kgs_ctx* ctx, int mode, int reps, double* ms_out) {
  if (!ctx || !ms_out || reps < 1) return fail(ctx, KGS_EINVAL, "bad arguments");
  Slab& s = ctx->slabs[0];
  PassGeom g = make_geom(ctx, s, 0, 0, s.nx);
  const int v = march_variant(ctx, s, g);
  if (v != 0 && v != 4) return fail(ctx, KGS_EINVAL, "debug pass needs march variant 0 or 4");
  if (int r0 = flush_pending(ctx)) return r0;
  Coeffs c{};
  CK(cudaSetDevice(s.dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int r = KGS_OK;
  for (int i = 0; i <= reps && !r; ++i) {
    if (i == 1) CK(cudaEventRecord(a, s.stream));
#define KGS_DBG(M)                                                                       \
  r = (v == 0) ? launch_march<MV0, 0, OP_BASE, OP_ADJ, false, false, M>(ctx, s, g, c, 0, v) \
               : launch_march<MV4, 0, OP_BASE, OP_ADJ, false, false, M>(ctx, s, g, c, 0, v);
    switch (mode) {
      case 0: KGS_DBG(0) break;
      case 1: KGS_DBG(1) break;
      default: KGS_DBG(3) break;
    }
#undef KGS_DBG
  }
  CK(cudaEventRecord(b, s.stream));
  CK(cudaEventSynchronize(b));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms_out = ms / reps;
  return r;
}

int kgs_selftest_division(int device, int64_t n, uint64_t seed, int64_t* mismatches) {
  kgs_ctx* ctx = nullptr;
  if (!mismatches || n < 0) return fail(nullptr, KGS_EINVAL, "bad arguments");
  CK(cudaSetDevice(device));
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, sizeof *d));
  CK(cudaMemset(d, 0, sizeof *d));
  division_selftest<<<1184, 256>>>(n, (unsigned long long)seed, d);
  cudaError_t e = cudaGetLastError();
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(nullptr, KGS_ECUDA, "division self-test: %s", cudaGetErrorString(e));
  *mismatches = (int64_t)h;
  return KGS_OK;
}

int kgs_set_promotion(kgs_ctx* ctx, int halo, int tile) {
  if (!ctx) return fail(nullptr, KGS_EINVAL, "ctx is NULL");
  ctx->tune_promo_halo = halo;
  ctx->tune_promo_tile = tile;
  for (auto& s : ctx->slabs) {
    if (ctx->d != 3) continue;
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.stream));
    int r = make_tensor_maps(ctx, s);
    if (r) return r;
  }
  return KGS_OK;
}

int kgs_set_param(kgs_ctx* ctx, const char* name, int value) {
  if (!ctx || !name) return fail(ctx, KGS_EINVAL, "NULL argument");
  const std::string n(name);
  if (n == "march_sync") ctx->tune_sync = std::max(1, value);
  else if (n == "march_variant") ctx->tune_variant = value;
  else if (n == "march_planes") ctx->tune_xc = value;
  else if (n == "blocks_per_sm") ctx->tune_occ = value;
  else if (n == "fused_step") ctx->tune_fused = value;
  else if (n == "fused_planes") ctx->tune_fused_xc = std::max(1, value);
  else if (n == "fused_debug") ctx->tune_fused_dbg = value;
  else if (n == "resident") ctx->tune_resident = value;
  else if (n == "tma_store") ctx->tune_tstore = value;
  else if (n == "pipeline") ctx->tune_pipe = value;
  else if (n == "pipeline_planes") ctx->tune_pipe_chunk = std::max(1, value);
  else if (n == "mirror_halo") ctx->tune_mirror = value;
  else return fail(ctx, KGS_EINVAL, "unknown tuning parameter '%s'", name);
  return KGS_OK;
}

int kgs_pass_timing(kgs_ctx* ctx, int enable) {
  if (!ctx) return fail(nullptr, KGS_EINVAL, "ctx is NULL");
  ctx->pass_timing = enable != 0;
  ctx->pass_count = 0;
  ctx->pass_ms = 0.0;
  ctx->pass_ev_used = 0;
  return KGS_OK;
}

int kgs_pass_stats(kgs_ctx* ctx, int64_t* launches, double* total_ms,
                   int64_t* points_per_launch) {
  if (!ctx) return fail(nullptr, KGS_EINVAL, "ctx is NULL");
  if (launches) *launches = ctx->pass_count;
  if (total_ms) *total_ms = ctx->pass_ms;
  if (points_per_launch) *points_per_launch = ctx->timed_pts;
  return KGS_OK;
}

int kgs_fill_preset(kgs_ctx* ctx, int preset) {
  if (!ctx) return fail(nullptr, KGS_EINVAL, "ctx is NULL");
  ctx->pending = false;  // the whole state is replaced
  const int need_d[4] = {3, 2, 2, 1};
  if (preset < 0 || preset > 3) return fail(ctx, KGS_EINVAL, "unknown preset %d", preset);
  if (need_d[preset] != ctx->d)
    return fail(ctx, KGS_EINVAL, "preset %d requires a %dD grid, got d=%d", preset,
                need_d[preset], ctx->d);
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    const int64_t n = (int64_t)s.nx * ctx->ny * ctx->nk * 2;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->nsm * 16);
    PassGeom g = make_geom(ctx, s, 0, 0, s.nx);   // own = black, oth = red
    fill_preset<<<blocks, 256, 0, s.stream>>>(g, ctx->a, ctx->h, preset);
    ctx->launches++;
    CK(cudaGetLastError());
  }
  ctx->mirrored[0] = ctx->mirrored[1] = false;  // planes written without mirroring
  int r = exchange(ctx, 0);
  if (!r) r = exchange(ctx, 1);
  if (!r) r = sync_all(ctx);
  return r;
}

}  // extern "C"
