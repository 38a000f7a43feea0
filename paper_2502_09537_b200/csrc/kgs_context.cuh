// kgs_context.cuh -- NCCL loader, slab and context state, error reporting, tile geometry.
// Part of the single translation unit kgs_host.cu (included in order).
#pragma once

namespace {

// march kernel variants (kgs_launch.cuh): MV0..MV15 (tile shapes, ring
// depths, rows per thread, clusters, producer warp); the default build
// compiles MV0, MV1 and MV4 (kVarBuilt), the others need -DKGS_EXPERIMENTAL
constexpr int kMarchVariantSlots = 16;

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
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
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
  KGS_SYM(AllReduce, "ncclAllReduce");
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
  MarchMaps maps[kMarchVariantSlots][2];  // [march variant][colour]: TMA descriptors
  bool has_tmaps[kMarchVariantSlots] = {};  // variant fits this geometry
  // fused steps (ping-pong): the other buffer set and its descriptors
  double* alt[2] = {nullptr, nullptr};
  double* alt0[2] = {nullptr, nullptr};
  MarchMaps amaps[kMarchVariantSlots][2];
#ifdef KGS_EXPERIMENTAL
  StepMaps smap[2];        // red of [0] the current set, [1] the other set
  bool has_smap = false;
#endif
  double* partials[2] = {nullptr, nullptr};  // per colour pass, grid * NTERMS
  int npart[2] = {0, 0};                     // blocks that wrote partials
  // record reductions run on their own stream (fstream), off the passes'
  // critical path: the partials are double-buffered per record (the set not
  // in use is partials_alt); fin_busy[s]: a reduction still reads set s,
  // done at ev_fin[s]; pset = the set `partials` points at
  double* partials_alt[2] = {nullptr, nullptr};
  cudaStream_t fstream = nullptr;
  cudaEvent_t ev_fin[2] = {nullptr, nullptr};
  cudaEvent_t ev_diag = nullptr;
  bool fin_busy[2] = {false, false};
  int pset = 0;
  double* records = nullptr;                 // device [cap * NTERMS]
  int64_t rec_cap = 0;
  unsigned long long* bad = nullptr;
  unsigned long long* wctr = nullptr;  // march wave-barrier arrivals (monotonic)
  unsigned long long wbase = 0;        // arrivals of all earlier launches
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
  cudaStream_t ustream = nullptr;   // uploads (off the comm stream: exchanges must not queue behind them)
  double* pipe_up = nullptr;        // natural-layout staging, one chunk of 4 fields
  double* pipe_dn = nullptr;
  int64_t pipe_stage = 0;           // doubles per staging buffer
  double* pipe_part = nullptr;      // per-record DIAG partials
  int64_t pipe_part_cap = 0;
  std::vector<cudaEvent_t> pipe_ev; // arrival / final events per chunk
  double* hslot = nullptr;          // page-locked host slots for pageable arrays
  int64_t hslot_len = 0;            // doubles per slot
  std::vector<cudaEvent_t> hslot_ev;  // last DMA of each slot
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
  // a 1-rank dist context that exchanges its faces with itself over NCCL
  // (KGS_SELF_EXCHANGE=1 test hook, kgs_create_dist): the multi-rank path on one GPU
  bool self_xch = false;
  ncclComm_t comm = nullptr;
  unsigned long long* dword = nullptr;   // device word for rank agreements (rank_min)
  std::string err = "no error";
  std::atomic<int64_t> launches{0};   // our kernel launches (the pipeline uploader thread adds too)
  double last_ms = 0.0;
  int nsm = 148;
  int grid_cap = 0;  // max persistent grid (blocks), sizes partials
  // tuning knobs (kgs_set_tuning): rows per tile, band height, blocks/SM cap
  int tune_ty = 4, tune_band_rows = 64, tune_occ = 0;
  int tune_gform = 2;  // record passes: gradient-term form (2 fast, 1 cancellation-free)
  int tune_sms = 0;  // march kernel: SMs its persistent grid spans (0: all)
  int tune_xc = 0;  // march kernel planes per unit (0 auto, < 0 disables it)
  int tune_variant = 4;  // march kernel variant (kgs_launch.cuh; MV4: 8 x 64 tiles, 2 rows per thread)
  int tune_promo_halo = 0, tune_promo_tile = 0;  // TMA L2 promotion (0 none .. 3 256B)
  int tune_sync = 4;     // march clusters: planes between cluster barriers
  int tune_wsync = 1;    // march: software grid barrier after every wave of units
  bool in_pipeline = false;  // kgs_integrate_host is issuing passes (wave barriers off)
  // deferred tail (KGS_STEP_DEFER_TAIL): the red adjoint of the last step is
  // pending and fuses with the next call's head when the coefficients match
  bool pending = false;
  Coeffs pend_c{};
  int tune_fused = 0;      // fused one-march DP-AVF2 steps (opt-in until faster)
  int tune_fused_xc = 128; // fused step: K4 planes per unit
  int tune_fused_dbg = 0;  // fused step timing experiments (results invalid)
  int tune_resident = 1;   // small grids: whole call in one launch (shared memory)
  int tune_tstore = 2;
  int tune_pdl = 1;          // colour passes: programmatic dependent launch
  int tune_pipe = 1;         // kgs_integrate_host: overlap upload | passes | download
  int tune_pipe_chunk = 0;   // planes per transfer chunk (0: auto, 16 or 32)
  int tune_stage = 1;        // kgs_integrate_host: stage pageable host arrays via page-locked slots     // march own-tile write: 0 STG, 1 TMA bulk store, 2 + L2 evict-first
  // fused halo exchange (single-process slabs): boundary launches
  // store their faces straight into the neighbours' ghost planes
  bool mirror = false;       // possible for this context (peer-accessible neighbours)
  int tune_mirror = 1;       // knob "mirror_halo"
  int64_t pass_no = 0;       // colour passes issued with the interior/boundary split
  bool mirrored[2] = {false, false};  // faces of colour c already in the ghosts
  bool alt_failed = false; // the second buffer set did not fit: two-pass steps
  bool backup_valid = false;  // the second buffer set holds a KGS_STEP_BACKUP copy
  int64_t timed_pts = 0;   // points updated twice per timed launch
  // per-pass timing (slab 0's stream): event pairs around fused passes
  bool pass_timing = false;
  std::vector<cudaEvent_t> pass_ev;
  size_t pass_ev_used = 0;
  int64_t pass_count = 0;
  double pass_ms = 0.0;
};

// Faces travel between slabs (several slabs, or ranks -- possibly one
// exchanging with itself); otherwise the single slab wraps in the kernel.
bool needs_exchange(const kgs_ctx* ctx) {
  return ctx->dist ? (ctx->nranks > 1 || ctx->self_xch) : ctx->slabs.size() > 1;
}

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
  g.wrap = needs_exchange(ctx) ? 0 : 1;
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
  g.fd_band = make_fastdiv((unsigned)std::max<int64_t>(1, (int64_t)(xb - xa) * nbt * g.nkt));
  g.fd_plane = make_fastdiv((unsigned)(nbt * g.nkt));
  g.fd_nkt = make_fastdiv((unsigned)g.nkt);
  g.fd_nk = make_fastdiv((unsigned)ctx->nk);
  g.fd_ny = make_fastdiv((unsigned)ctx->ny);
  return g;
}

}  // namespace
