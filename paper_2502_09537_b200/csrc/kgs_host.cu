// kgs_host.cu -- C ABI (include/kgs_b200.h) over the sm_100a colour-pass
// kernels: contexts, state transfer, the DP-AVF2 stepping loop, diagnostics.
// One translation unit; the host runtime is split by concern into
//   kgs_context.cuh   NCCL loader, slab / context state, errors, geometry
//   kgs_launch.cuh    kernel dispatch (simple / marching / resident / fused)
//   kgs_passes.cuh    colour passes over all slabs, halo exchange, records
//   kgs_pipeline.cuh  pipelined host integration (kgs_integrate_host)
// and kgs_device.cuh holds the device code.  See DESIGN.md for the pass
// schedule and the rooflines.
#include "../../include/kgs_b200.h"
#include "kgs_device.cuh"

#include <dlfcn.h>
#include <immintrin.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <climits>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace kgs;

#include "kgs_context.cuh"
#include "kgs_launch.cuh"
#include "kgs_program.cuh"
#include "kgs_passes.cuh"
#ifdef KGS_EXPERIMENTAL
#include "kgs_exp_step.cuh"
#endif

// =========================================================================
// extern "C" API
// =========================================================================
extern "C" {

int kgs_abi_version(void) { return 102; }

int kgs_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int kgs_build_flags(void) {
  int f = 0;
#ifdef KGS_EXPERIMENTAL
  f |= KGS_BUILD_EXPERIMENTAL;
#endif
#ifdef KGS_CHECKED
  f |= KGS_BUILD_CHECKED;
#endif
  return f;
}

const char* kgs_last_error(kgs_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

int64_t kgs_launch_count(kgs_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

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
  if (nranks == 1 && nccl_id) {
    const char* e = std::getenv("KGS_SELF_EXCHANGE");
    ctx->self_xch = e && e[0] == '1';
  }
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
  if (!r && (nranks > 1 || ctx->self_xch)) {
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
  if (ctx->dword) {
    cudaSetDevice(ctx->slabs.empty() ? 0 : ctx->slabs[0].dev);
    cudaFree(ctx->dword);
  }
  for (auto e : ctx->pass_ev) cudaEventDestroy(e);
  for (auto& s : ctx->slabs) {
    cudaSetDevice(s.dev);
    if (s.stream) cudaStreamSynchronize(s.stream);
    if (s.fstream) cudaStreamSynchronize(s.fstream);
    for (int c = 0; c < 2; ++c) {
      if (s.buf[c]) cudaFree(s.buf[c]);
      if (s.partials[c]) cudaFree(s.partials[c]);
      if (s.partials_alt[c]) cudaFree(s.partials_alt[c]);
    }
    for (int i = 0; i < 2; ++i)
      if (s.ev_fin[i]) cudaEventDestroy(s.ev_fin[i]);
    if (s.ev_diag) cudaEventDestroy(s.ev_diag);
    if (s.fstream) cudaStreamDestroy(s.fstream);
    if (s.records) cudaFree(s.records);
    if (s.bad) cudaFree(s.bad);
    if (s.wctr) cudaFree(s.wctr);
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
    if (s.ustream) cudaStreamSynchronize(s.ustream);
    for (auto e : s.pipe_ev) cudaEventDestroy(e);
    for (auto e : s.hslot_ev) cudaEventDestroy(e);
    if (s.hslot) cudaFreeHost(s.hslot);
    if (s.dstream) cudaStreamDestroy(s.dstream);
    if (s.ustream) cudaStreamDestroy(s.ustream);
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

}  // namespace

#include "kgs_pipeline.cuh"

namespace {

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
  ctx->backup_valid = false;
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
  if (r) return r;
  ctx->backup_valid = false;
  r = flush_pending(ctx);
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
  ctx->backup_valid = false;
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
  ctx->backup_valid = false;
  if (flags & KGS_STEP_BACKUP) {
    // the state at step_offset (a pending tail applied first) into the
    // second buffer set, ghosts included, for kgs_restore_backup
    r = flush_pending(ctx);
    if (!r && ensure_alt(ctx) == KGS_OK) {
      for (auto& s : ctx->slabs) {
        CK(cudaSetDevice(s.dev));
        for (int cc = 0; cc < 2; ++cc)
          CK(cudaMemcpyAsync(s.alt[cc], s.buf[cc], (size_t)(s.nx + 2) * ctx->ps * 8,
                             cudaMemcpyDeviceToDevice, s.stream));
      }
      ctx->backup_valid = true;
    }
    if (r) return r;
  }
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaEventRecord(s.ev_t0, s.stream));
  }
  const int64_t last = step_offset + nsteps;
  const bool defer = (flags & KGS_STEP_DEFER_TAIL) &&
                     !(record_stride > 0 && last % record_stride == 0);
  const bool resident = resident_eligible(ctx);
  // head: base red(first step) -- fused with a deferred red adjoint of the
  // previous call when its coefficients are the same (bitwise neutral);
  // a pending adjoint with other coefficients is applied first
  const bool head_fused = ctx->pending && std::memcmp(&ctx->pend_c, &c, sizeof c) == 0;
  if (head_fused) ctx->pending = false;
  else r = flush_pending(ctx);
#ifdef KGS_EXPERIMENTAL
  const bool fused = !resident && fused_ready(ctx);
#else
  constexpr bool fused = false;
#endif
  if (r) {
  } else if (resident) {
    // the whole call in one launch (state in shared memory)
    r = launch_resident(ctx, c, nsteps, step_offset, record_stride, head_fused, defer);
    if (!r && defer) {
      ctx->pending = true;
      ctx->pend_c = c;
    }
  } else if (!fused) {
    // the pass program (kgs_program.cuh): head, K3/K4 per step, exchanges,
    // records, deferred tail -- the same list kgs_step_program exports
    const Program prog = step_program(ctx->slabs[0].nx, needs_exchange(ctx), nsteps,
                                      step_offset, record_stride,
                                      (head_fused ? PGF_HEAD_FUSED : 0) |
                                          ((flags & KGS_STEP_DEFER_TAIL) ? PGF_DEFER : 0));
    r = run_program(ctx, prog, c);
  }
#ifdef KGS_EXPERIMENTAL
  else {
    r = step_loop_fused(ctx, c, nsteps, step_offset, record_stride, head_fused, defer);
  }
#endif
  if (r) return r;
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    // the step ends when the last halo exchange has landed
    if (s.xch_pending) CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
    // ... and its record reductions (record stream) are done
    for (int i = 0; i < 2; ++i)
      if (s.fin_busy[i]) CK(cudaStreamWaitEvent(s.stream, s.ev_fin[i], 0));
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

int kgs_restore_backup(kgs_ctx* ctx) {
  if (!ctx) return fail(nullptr, KGS_EINVAL, "ctx is NULL");
  if (!ctx->backup_valid)
    return fail(ctx, KGS_EINVAL, "no backup: the last kgs_step_dpavf2 call had no "
                "KGS_STEP_BACKUP (or no memory for it), or the state changed since");
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.cstream));
    for (int cc = 0; cc < 2; ++cc)
      CK(cudaMemcpyAsync(s.buf[cc], s.alt[cc], (size_t)(s.nx + 2) * ctx->ps * 8,
                         cudaMemcpyDeviceToDevice, s.stream));
    s.xch_pending = false;
  }
  ctx->pending = false;                          // the backup is a complete state
  ctx->mirrored[0] = ctx->mirrored[1] = false;   // ghosts restored with it
  ctx->backup_valid = false;
  return sync_all(ctx);
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

int64_t kgs_step_program(int64_t nx, int split, int64_t nsteps, int64_t step_offset,
                         int64_t record_stride, int flags, int64_t* out, int64_t cap) {
  if (nx < 1 || (split && nx < 2) || nsteps < 0 || step_offset < 0 || record_stride < 0 ||
      nsteps + step_offset > INT_MAX || cap < 0 || (cap > 0 && !out))
    return -1;
  const Program p = step_program(nx, split != 0, nsteps, step_offset, record_stride,
                                 ((flags & KGS_PROGRAM_HEAD_FUSED) ? PGF_HEAD_FUSED : 0) |
                                     ((flags & KGS_STEP_DEFER_TAIL) ? PGF_DEFER : 0));
  const int64_t n = (int64_t)p.size();
  for (int64_t i = 0; i < std::min(n, cap); ++i) {
    const ProgOp& o = p[i];
    const int64_t row[kProgFields] = {o.kind, o.col, o.op1, o.op2, o.diag, o.check, o.step,
                                      o.xa, o.xb};
    std::copy(row, row + kProgFields, out + kProgFields * i);
  }
  return n;
}

int64_t kgs_pipeline_plan(int64_t N, int64_t C, int64_t nsteps, int split, int64_t* out,
                          int64_t cap) {
  if (N < 1 || C < 1 || nsteps < 0 || cap < 0 || (cap > 0 && !out)) return -1;
  const std::vector<char> writes = pipeline_writes(nsteps);
  const std::vector<PipeEvent> plan =
      pipeline_plan(N, C, pipeline_shrinks(nsteps), split ? &writes : nullptr);
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
  ctx->backup_valid = false;   // the pipeline uses the second buffer set itself
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
    unsigned long long b = r == KGS_ENONFINITE ? (unsigned long long)fb : ULLONG_MAX;
    if (int e = rank_min(ctx, &b)) return e;   // the ranks replay to the same step
    fb = (int64_t)b;
    if (b != ULLONG_MAX) {   // replay from the (untouched) host state to the bad step
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
  std::vector<double> rec((size_t)(nrec + 1) * NTERMS), tmp(rec.size());
  for (auto& s : ctx->slabs) {   // slab order: deterministic host sum (as kgs_step_dpavf2)
    CK(cudaSetDevice(s.dev));
    CK(cudaMemcpy(tmp.data(), s.records, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (size_t q = 0; q < rec.size(); ++q) rec[q] += tmp[q];
  }
  std::copy(rec.begin(), rec.begin() + NTERMS, terms0);
  if (nrec > 0) std::copy(rec.begin() + NTERMS, rec.end(), terms_out);
  if (bad != ULLONG_MAX) {
    // restore the initial state (device copy) and replay exactly to the bad step
    // (on the slab stream: a device-to-device cudaMemcpy would not order
    // itself before the replay's kernels on this non-blocking stream); the
    // copy holds no ghost planes, so several slabs exchange their faces first
    for (auto& s : ctx->slabs) {
      CK(cudaSetDevice(s.dev));
      for (int cc = 0; cc < 2; ++cc)
        CK(cudaMemcpyAsync(s.buf[cc], s.alt[cc], (size_t)(s.nx + 2) * ctx->ps * 8,
                           cudaMemcpyDeviceToDevice, s.stream));
    }
    r = exchange(ctx, 0);
    if (!r) r = exchange(ctx, 1);
    if (r) return r;
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
#ifndef KGS_EXPERIMENTAL
  (void)mode;
  return fail(ctx, KGS_EINVAL, "kgs_debug_pass needs a -DKGS_EXPERIMENTAL build "
              "(python -m paper_2502_09537_b200.build --experimental)");
#else
  Slab& s = ctx->slabs[0];
  PassGeom g = make_geom(ctx, s, 0, 0, s.nx);
  const int v = march_variant(ctx, s, g);
  if (v != 0 && v != 4 && v != 13)
    return fail(ctx, KGS_EINVAL, "debug pass needs march variant 0, 4 or 13");
  if (int r0 = flush_pending(ctx)) return r0;
  Coeffs c{};
  CK(cudaSetDevice(s.dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  if (cudaEventCreate(&b) != cudaSuccess) {
    cudaEventDestroy(a);
    return fail(ctx, KGS_ECUDA, "cudaEventCreate failed");
  }
  int r = KGS_OK;
  for (int i = 0; i <= reps && !r; ++i) {
    if (i == 1) CK(cudaEventRecord(a, s.stream));
#define KGS_DBG(M)                                                                         \
  r = (v == 0)   ? launch_march<MV0, 0, OP_BASE, OP_ADJ, false, false, M>(ctx, s, g, c, 0, v)  \
      : (v == 4) ? launch_march<MV4, 0, OP_BASE, OP_ADJ, false, false, M>(ctx, s, g, c, 0, v)  \
                 : launch_march<MV13, 0, OP_BASE, OP_ADJ, false, false, M>(ctx, s, g, c, 0, v);
    switch (mode) {
      case 0: KGS_DBG(0) break;
      case 1: KGS_DBG(1) break;
      case 4: KGS_DBG(4) break;
      case 5: KGS_DBG(5) break;
      default: KGS_DBG(3) break;
    }
#undef KGS_DBG
  }
  float ms = 0.f;
  cudaError_t e = cudaSuccess;
  if (!r) e = cudaEventRecord(b, s.stream);
  if (!r && e == cudaSuccess) e = cudaEventSynchronize(b);
  if (!r && e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (r) return r;
  if (e != cudaSuccess) return fail(ctx, KGS_ECUDA, "debug pass: %s", cudaGetErrorString(e));
  *ms_out = ms / reps;
  return KGS_OK;
#endif
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
  else if (n == "march_wave_sync") ctx->tune_wsync = value;
  else if (n == "march_variant") {
    if (value >= kMarchVariantSlots || (value >= 0 && !kVarBuilt[value]))
      return fail(ctx, KGS_EINVAL, "march_variant %d not in this build (default build: 0, 1, "
                  "4; the others need -DKGS_EXPERIMENTAL)", value);
    ctx->tune_variant = value;
  }
  else if (n == "march_planes") ctx->tune_xc = value;
  else if (n == "blocks_per_sm") ctx->tune_occ = value;
  else if (n == "march_sms") ctx->tune_sms = value;
  else if (n == "record_form") {
    if (value != 1 && value != 2)
      return fail(ctx, KGS_EINVAL, "record_form must be 1 (differences) or 2 (sums of squares)");
    ctx->tune_gform = value;
  }
  else if (n == "fused_step") {
#ifndef KGS_EXPERIMENTAL
    if (value) return fail(ctx, KGS_EINVAL, "fused_step needs a -DKGS_EXPERIMENTAL build");
#endif
    ctx->tune_fused = value;
  }
  else if (n == "fused_planes") ctx->tune_fused_xc = std::max(1, value);
  else if (n == "fused_debug") ctx->tune_fused_dbg = value;
  else if (n == "resident") ctx->tune_resident = value;
  else if (n == "tma_store") ctx->tune_tstore = value;
  else if (n == "pipeline") ctx->tune_pipe = value;
  else if (n == "pipeline_planes") ctx->tune_pipe_chunk = std::max(0, value);   // 0: auto
  else if (n == "stage_pageable") ctx->tune_stage = value;
  else if (n == "mirror_halo") ctx->tune_mirror = value;
  else if (n == "pdl") ctx->tune_pdl = value;
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
  ctx->backup_valid = false;
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
