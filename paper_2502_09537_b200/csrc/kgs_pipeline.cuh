// kgs_pipeline.cuh -- pipelined host integration (kgs_integrate_host):
// the wavefront plan and its execution.
// Part of the single translation unit kgs_host.cu (included in order).
#pragma once

namespace {

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
// H2D, compute and D2H proceed together (pinned copies: 55-57 GB/s one way,
// 46 GB/s each way when both run).  After the last chunk, a pass whose
// predecessor has the whole ring grows by one chunk per side per round, so
// the remaining gap closes from its edges and those blocks go back while the
// middle still computes.  The initial
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
        for (int cc = 0; cc < 2; ++cc) {   // do not hold half a buffer set
          if (s.alt[cc]) cudaFree(s.alt[cc]);
          s.alt[cc] = s.alt0[cc] = nullptr;
        }
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
// over planes [a, b)), FINAL (planes [a, b) are final: copy them back),
// XCH (several slabs / ranks: exchange the faces pass j wrote; j = -1: both
// colours' faces of the arrived state).
// Pure host logic (kgs_pipeline_plan exports it for the CPU tests).
//
// Several slabs (`writes` given): every slab runs the same plan on its own
// planes, so a slab's local plane -1 (unwrapped) is its lower neighbour's
// plane nx-1, which that neighbour covers at the same point of the same plan
// -- the done regions are intervals around every slab boundary, and a pass
// reads its ghost planes only in launches covering plane 0 or nx-1.  So a
// writing pass's faces are exchanged as soon as it has covered both
// boundary planes (before any launch of its successor can reach them, which
// needs exactly that coverage), and a launch covering a boundary plane
// waits for the pending exchange.  The arrived state's faces are exchanged
// once both boundary blocks are in (the first two chunks, folded order).
enum PipeKind : int { PIPE_ARRIVE = 0, PIPE_PASS = 1, PIPE_FINAL = 2, PIPE_XCH = 3 };
struct PipeEvent {
  int kind, pass;
  int64_t a, b;
};

std::vector<PipeEvent> pipeline_plan(int64_t N, int64_t C, const std::vector<int>& shrink,
                                     const std::vector<char>* writes = nullptr) {
  std::vector<PipeEvent> ev;
  const int64_t nb = (N + C - 1) / C;
  const int J = (int)shrink.size();
  std::vector<int64_t> lo(J, 0), hi(J, 0);   // done regions, unwrapped: empty or lo < hi
  std::vector<char> dl(nb, 0), xch(J, 0);
  // unwrapped region of pass j contains plane x (or the whole ring)
  auto covers = [&](int j, int64_t x) {
    return hi[j] - lo[j] >= N || (lo[j] <= x && x < hi[j]) || (lo[j] <= x - N && x - N < hi[j]);
  };
  auto exchange_after = [&](int j) {   // pass j's faces, once both boundary planes are done
    if (writes && (*writes)[j] && !xch[j] && covers(j, 0) && covers(j, N - 1)) {
      xch[j] = 1;
      ev.push_back({PIPE_XCH, j, 0, 0});
    }
  };
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
  auto full = [&](int j) { return hi[j] - lo[j] >= N; };
  // One round: every pass extends its done region as far as its predecessor
  // allows -- the predecessor's region shrunk by `shrink` planes per side; once
  // the predecessor has the whole ring, by at most C planes per side, so the
  // last planes close from both edges inward and blocks near the edges
  // become final (and go back) while the middle still computes.
  auto round = [&](int64_t alo, int64_t ahi) {
    int64_t plo = alo, phi = ahi;
    for (int j = 0; j < J; ++j) {
      if (!full(j)) {
        if (phi - plo >= N) {                   // predecessor complete
          if (lo[j] == hi[j]) { pass(j, 0, N); lo[j] = 0; hi[j] = N; }
          else {
            const int64_t gap = N - (hi[j] - lo[j]);
            const int64_t r = std::min(C, gap), l = std::min(C, gap - r);
            pass_u(j, hi[j], hi[j] + r);
            pass_u(j, lo[j] - l, lo[j]);
            hi[j] += r;
            lo[j] -= l;
          }
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
      exchange_after(j);
      plo = lo[j];
      phi = hi[j];
    }
    // blocks wholly inside the last pass's done region (which need not
    // contain plane 0) are final
    const int64_t L = lo[J - 1], H = hi[J - 1];
    for (int64_t k = 0; k < nb; ++k) {
      if (dl[k]) continue;
      const int64_t b0 = k * C, b1 = std::min(N, b0 + C);
      if (full(J - 1) || (L < H && ((b0 >= L && b1 <= H) || (b0 - N >= L && b1 - N <= H)))) {
        dl[k] = 1;
        ev.push_back({PIPE_FINAL, (int)k, b0, b1});
      }
    }
  };
  int64_t alo = 0, ahi = 0;
  for (int64_t m = 0; m < nb; ++m) {
    const int64_t blk = (m % 2 == 0) ? m / 2 : nb - 1 - m / 2;   // folded order
    const int64_t x0 = blk * C, x1 = std::min(N, x0 + C);
    ev.push_back({PIPE_ARRIVE, (int)m, x0, x1});
    if (m % 2 == 0) ahi = x1; else alo = x0 - N;
    if (m == nb - 1) { alo = 0; ahi = N; }       // the whole ring has arrived
    if (writes && m == std::min<int64_t>(1, nb - 1))   // blocks 0 and nb-1 are in
      ev.push_back({PIPE_XCH, -1, 0, 0});
    round(alo, ahi);
  }
  for (int guard = 0; !full(J - 1) && guard < 4 * (int)nb + J + 4; ++guard) round(0, N);
  return ev;
}

std::vector<int> pipeline_shrinks(int64_t nsteps) {
  // initial energy (black self, red edges + self), head, then K3/K4 per step
  std::vector<int> sh = {0, 1, 0};
  for (int64_t i = 0; i < 2 * nsteps; ++i) sh.push_back(1);
  return sh;
}

std::vector<char> pipeline_writes(int64_t nsteps) {
  // the energy passes only read; the head and every K3/K4 write their colour
  std::vector<char> w = {0, 0, 1};
  for (int64_t i = 0; i < 2 * nsteps; ++i) w.push_back(1);
  return w;
}

// ---- pageable host arrays: page-locked bounce slots ---------------------
// The reference's FieldState holds ordinary numpy arrays (grid.py:82-103):
// pageable memory, which cudaMemcpyAsync copies through a small driver
// buffer synchronously (~11 GB/s measured), and page-locking them in place
// (cudaHostRegister) runs at only 6-14 GB/s and does not scale with threads
// (tools/pageable_probe.py).  So for pageable arrays the
// pipeline stages every chunk through page-locked slots of its own: an
// uploader thread copies chunk m into an upload slot with a team of host
// threads and queues the DMA from it; a downloader thread copies each
// finished block out of a download slot once its DMA has landed.  The
// device side (arrival events, passes, merges) is unchanged.
constexpr int kUpSlots = 2, kDnSlots = 3;

bool host_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Copy with non-temporal (streaming) stores: the destination is not read
// for ownership, so a staged byte costs one host-memory read and one write
// instead of two reads and a write (host bandwidth is the bottleneck of a
// staged transfer: every byte is also read or written once more by the DMA).
__attribute__((target("avx512f"))) void stream_copy_avx512(char* dst, const char* src,
                                                           size_t n) {
  size_t head = (64 - ((uintptr_t)dst & 63)) & 63;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  const size_t body = n & ~(size_t)255;
  for (size_t i = 0; i < body; i += 256) {
    const __m512i a = _mm512_loadu_si512((const void*)(src + i));
    const __m512i b = _mm512_loadu_si512((const void*)(src + i + 64));
    const __m512i c = _mm512_loadu_si512((const void*)(src + i + 128));
    const __m512i d = _mm512_loadu_si512((const void*)(src + i + 192));
    _mm512_stream_si512((__m512i*)(dst + i), a);
    _mm512_stream_si512((__m512i*)(dst + i + 64), b);
    _mm512_stream_si512((__m512i*)(dst + i + 128), c);
    _mm512_stream_si512((__m512i*)(dst + i + 192), d);
  }
  _mm_sfence();
  std::memcpy(dst + body, src + body, n - body);
}

void stream_copy(char* dst, const char* src, size_t n) {
  static const bool avx512 = __builtin_cpu_supports("avx512f");
  if (avx512 && n >= 4096) stream_copy_avx512(dst, src, n);
  else std::memcpy(dst, src, n);
}

// stream_copy with `threads` host threads (page-sized parts)
void par_copy(char* dst, const char* src, size_t n, int threads) {
  if (threads <= 1 || n < ((size_t)8 << 20)) {
    stream_copy(dst, src, n);
    return;
  }
  const size_t part = ((n + threads - 1) / threads + 4095) & ~(size_t)4095;
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t) {
    const size_t lo = (size_t)t * part;
    if (lo >= n) break;
    th.emplace_back([=] { stream_copy(dst + lo, src + lo, std::min(part, n - lo)); });
  }
  for (auto& x : th) x.join();
}

// Page-locked slots of `slot` doubles each (cached in the slab).
int ensure_host_slots(kgs_ctx* ctx, Slab& s, int64_t slot) {
  const int n = kUpSlots + kDnSlots;
  if (s.hslot && s.hslot_len >= slot) return KGS_OK;
  if (s.hslot) cudaFreeHost(s.hslot);
  s.hslot = nullptr;
  s.hslot_len = 0;
  if (cudaHostAlloc(&s.hslot, (size_t)(n * slot) * 8, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    s.hslot = nullptr;
    return KGS_ENOMEM;
  }
  s.hslot_len = slot;
  while ((int)s.hslot_ev.size() < n) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s.hslot_ev.push_back(e);
  }
  return KGS_OK;
}

int integrate_pipelined(kgs_ctx* ctx, double* const host[4], const Coeffs& c, int64_t nsteps,
                        int64_t step_offset, int64_t record_stride, int64_t nrec,
                        unsigned long long* bad_out) {
  const int ns = (int)ctx->slabs.size();
  // several slabs / ranks: every slab runs the same plan on its own planes,
  // with face exchanges between the passes (pipeline_plan)
  const bool split = needs_exchange(ctx);
  const int64_t N = ctx->slabs[0].nx;   // planes per slab
  // pageable arrays (the reference's numpy FieldState): staged through
  // page-locked slots by host threads (one ring of slots for all slabs);
  // page-locked arrays (FieldState.pinned) go direct.
  bool staged = false;
  if (ctx->tune_stage)
    for (int f = 0; f < 4; ++f) staged = staged || host_pageable(host[f]);
  // doubles of per-record partials for chunks of c planes: every launch of
  // a pass (<= chunks + 4) writes grid_cap blocks of NTERMS, per record and colour
  auto partials_for = [&](int64_t c) {
    return (nrec + 1) * 2 * (((N + c - 1) / c + 4) * ctx->grid_cap * NTERMS);
  };
  constexpr int64_t kPartMax = (int64_t)1 << 27;               // 1 GiB of partials per slab
  // chunk planes (knob pipeline_planes; 0 = auto: 16 for page-locked arrays
  // -- the shorter wavefront drain; 1024^3, 20 steps: 0.848 vs 0.877 s per
  // call -- unless that many partial regions do not fit, else 32); a
  // layout-transform launch covers < 2^31 point pairs (decode_point)
  int64_t want = ctx->tune_pipe_chunk;
  if (want <= 0) want = (!staged && partials_for(16) <= kPartMax) ? 16 : 32;
  const int64_t C = std::max<int64_t>(1, std::min<int64_t>(want,
                                                           ((1ll << 31) - 1) / ((int64_t)ctx->ny * ctx->nk)));
  const int64_t nb = (N + C - 1) / C;
  const int64_t nat_plane = (int64_t)ctx->ny * ctx->nz;
  const int64_t stage = 4 * C * nat_plane;
  const int64_t maxl = nb + 4;                                 // launches per pass
  const int64_t region = maxl * ctx->grid_cap * NTERMS;        // doubles per (record, colour)
  const int64_t need = (nrec + 1) * 2 * region;
  // eligibility and buffers; the ranks of a torchrun job then agree, so all
  // of them run the pipeline (with its exchanges) or none does
  auto prepare = [&]() -> int {
    if (!ctx->tune_pipe || ctx->d != 3 || nb < 4) return kPipeFallback;
    for (const Slab& s : ctx->slabs)
      if (s.nx != N) return kPipeFallback;
    if (need > kPartMax) return kPipeFallback;
    if (ensure_alt(ctx)) return kPipeFallback;
    for (Slab& s : ctx->slabs) {
      CK(cudaSetDevice(s.dev));
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
      if (s.pipe_part_cap < need) {
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
      if (!s.ustream) CK(cudaStreamCreateWithFlags(&s.ustream, cudaStreamNonBlocking));
      while ((int64_t)s.pipe_ev.size() < 2 * nb) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s.pipe_ev.push_back(e);
      }
    }
    return KGS_OK;
  };
  const int pr = prepare();
  unsigned long long go = pr == KGS_OK ? 1 : 0;
  if (int e = rank_min(ctx, &go)) return e;
  if (pr) return pr;                  // an error, or this rank's fallback
  if (!go) return kPipeFallback;      // another rank cannot run it
  int r = ensure_records(ctx, nrec + 1);
  if (!r) r = reset_bad(ctx);
  if (r) return r;
  ctx->pending = false;   // the whole state is replaced
  // the ghost planes are filled by this call's own exchanges
  ctx->mirrored[0] = ctx->mirrored[1] = false;
  for (Slab& s : ctx->slabs) s.xch_pending = false;

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
  std::vector<int> shrink(J);
  for (int j = 0; j < J; ++j) shrink[j] = passes[j].shrink;
  const std::vector<char> writes = pipeline_writes(nsteps);
  const std::vector<PipeEvent> plan = pipeline_plan(N, C, shrink, split ? &writes : nullptr);
  // partials written so far per (slab, record, colour)
  std::vector<std::vector<int64_t>> roff(ns, std::vector<int64_t>((size_t)(nrec + 1) * 2, 0));

  // the passes run next to the transfer streams' kernels: no wave barriers
  struct PipeFlag {
    kgs_ctx* c;
    ~PipeFlag() { c->in_pipeline = false; }
  } pipe_flag{ctx};
  ctx->in_pipeline = true;
  auto launch_range = [&](int si, const PipePass& P, int64_t xa, int64_t xb) -> int {
    if (xb <= xa) return KGS_OK;
    Slab& s = ctx->slabs[si];
    CK(cudaSetDevice(s.dev));
    if (s.xch_pending && (xa == 0 || xb == s.nx)) {   // reads the ghost planes
      CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
      s.xch_pending = false;
    }
    double* save = s.partials[P.col];
    const int64_t ri = P.diag ? (int64_t)P.rec * 2 + P.col : 0;
    if (P.diag) {
      s.partials[P.col] = s.pipe_part + ri * region;
      s.npart[P.col] = (int)roff[si][ri];
    }
    int rr = launch_pass(ctx, s, P.col, P.op1, P.op2, P.diag, P.check, c, P.step_no, (int)xa,
                         (int)xb);
    if (P.diag) {
      roff[si][ri] = s.npart[P.col];
      s.partials[P.col] = save;
    }
    return rr;
  };

  Slab& s0 = ctx->slabs[0];
  if (staged && ensure_host_slots(ctx, s0, stage) != KGS_OK) staged = false;
  if (staged)   // slot events of every slab, on its own device (slab 0's come with the slots)
    for (Slab& s : ctx->slabs) {
      CK(cudaSetDevice(s.dev));
      while ((int)s.hslot_ev.size() < kUpSlots + kDnSlots) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s.hslot_ev.push_back(e);
      }
    }
  // host threads per direction (uploads and downloads copy concurrently)
  const int cp_threads = std::max(1, std::min(8, ((int)std::thread::hardware_concurrency() - 2) / 2));
  auto up_slot = [&](int64_t u) { return s0.hslot + (u % kUpSlots) * stage; };
  // upload slot uses in issue order (chunk-major, slab-minor) and, per slot,
  // the event of its last DMA (on that slab's upload stream)
  int64_t up_idx = 0;
  cudaEvent_t last_up[kUpSlots] = {};
  // KGS_PIPE_DEBUG=1: host-side time breakdown of a staged call on stderr
  static const bool dbg = std::getenv("KGS_PIPE_DEBUG") != nullptr;
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  const clk::time_point t_call = clk::now();
  double up_wait = 0, up_copy = 0, dn_wait = 0, dn_copy = 0, main_wait_up = 0, main_wait_dn = 0;
  auto dn_slot = [&](int64_t j) { return s0.hslot + (kUpSlots + j % kDnSlots) * stage; };

  CK(cudaSetDevice(s0.dev));
  CK(cudaEventRecord(s0.ev_t0, s0.stream));
  for (Slab& s : ctx->slabs) {   // uploads start after the call does
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamWaitEvent(s.ustream, s0.ev_t0, 0));
  }
  // uploads (folded block order) on the upload stream: H2D, split, backup
  // copy.  The host arrays hold this context's planes (kgs_upload's
  // convention: the whole grid, or a rank's slab), slab s from s.x0 - hx0 on.
  int64_t hx0 = 0;
  kgs_local_range(ctx, &hx0, nullptr, nullptr);
  auto upload_chunk = [&](Slab& s, const PipeEvent& e) -> int {
    const int64_t m = e.pass, x0 = e.a, x1 = e.b, nxc = x1 - x0;
    const int64_t gx = s.x0 - hx0 + x0;
    const size_t bytes = (size_t)nxc * nat_plane * 8;
    CK(cudaSetDevice(s.dev));
    if (staged) {
      const int64_t u = up_idx++;
      const int k = (int)(u % kUpSlots);
      const clk::time_point t0 = clk::now();
      if (last_up[k]) CK(cudaEventSynchronize(last_up[k]));   // the slot's last DMA has read it
      const clk::time_point t1 = clk::now();
      double* sl = up_slot(u);
      for (int f = 0; f < 4; ++f)
        par_copy((char*)(sl + f * C * nat_plane), (const char*)(host[f] + gx * nat_plane), bytes,
                 cp_threads);
      up_wait += secs(t0, t1);
      up_copy += secs(t1, clk::now());
      for (int f = 0; f < 4; ++f)
        CK(cudaMemcpyAsync(s.pipe_up + f * C * nat_plane, sl + f * C * nat_plane, bytes,
                           cudaMemcpyHostToDevice, s.ustream));
      CK(cudaEventRecord(s.hslot_ev[k], s.ustream));
      last_up[k] = s.hslot_ev[k];
    } else {
      for (int f = 0; f < 4; ++f)
        CK(cudaMemcpyAsync(s.pipe_up + f * C * nat_plane, host[f] + gx * nat_plane, bytes,
                           cudaMemcpyHostToDevice, s.ustream));
    }
    const int64_t cnt = nxc * ctx->ny * ctx->nk;
    const int blocks = (int)std::min<int64_t>((cnt + 255) / 256, (int64_t)ctx->nsm * 16);
    for (int f = 0; f < 4; ++f) {
      PassGeom g = make_geom(ctx, s, 1, 0, s.nx);   // own = red, oth = black
      g.own += f * ctx->pp;
      g.oth += f * ctx->pp;
      split_field<<<blocks, 256, 0, s.ustream>>>(s.pipe_up + f * C * nat_plane, g, (int)nxc,
                                                   (int)x0);
      ctx->launches++;
    }
    CK(cudaGetLastError());
    for (int cc = 0; cc < 2; ++cc)
      CK(cudaMemcpyAsync(s.alt0[cc] + x0 * ctx->ps, s.plane0[cc] + x0 * ctx->ps,
                         (size_t)nxc * ctx->ps * 8, cudaMemcpyDeviceToDevice, s.ustream));
    CK(cudaEventRecord(s.pipe_ev[m], s.ustream));
    return KGS_OK;
  };

  // staged: an uploader thread stages and queues the chunks (the passes
  // below wait, host side, until a chunk's arrival event is recorded before
  // queueing a wait on it); a downloader thread empties the download slots
  std::mutex mu;
  std::condition_variable cv;
  int64_t arrived = 0;          // chunks whose arrival event is recorded
  int err = KGS_OK;             // first error of a helper thread
  struct DlJob { int64_t b0, nxc, j; int si; };
  std::vector<DlJob> dl_queue;  // download slot jobs, in issue order
  size_t dl_next = 0;           // next job for the downloader
  int64_t dl_done = 0;          // jobs whose host copy finished
  bool dl_close = false;
  std::thread uploader, downloader;
  if (staged) {
    uploader = std::thread([&] {
      cudaSetDevice(s0.dev);
      for (const PipeEvent& e : plan) {
        if (e.kind != PIPE_ARRIVE) continue;
        int rc = KGS_OK;
        for (Slab& s : ctx->slabs)
          if (!rc) rc = upload_chunk(s, e);
        {
          std::lock_guard<std::mutex> lk(mu);
          if (rc && !err) err = rc;
          arrived = e.pass + 1;
        }
        cv.notify_all();
        if (rc) break;
      }
    });
    downloader = std::thread([&] {
      cudaSetDevice(s0.dev);
      for (;;) {
        DlJob jb;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return dl_next < dl_queue.size() || dl_close; });
          if (dl_next >= dl_queue.size()) return;
          jb = dl_queue[dl_next++];
        }
        const clk::time_point t0 = clk::now();
        const Slab& sj = ctx->slabs[jb.si];
        int rc = cudaEventSynchronize(sj.hslot_ev[kUpSlots + jb.j % kDnSlots]) == cudaSuccess
                     ? KGS_OK : fail(ctx, KGS_ECUDA, "download slot event failed");
        const clk::time_point t1 = clk::now();
        if (!rc) {
          const double* sl = dn_slot(jb.j);
          for (int f = 0; f < 4; ++f)
            par_copy((char*)(host[f] + (sj.x0 - hx0 + jb.b0) * nat_plane),
                     (const char*)(sl + f * C * nat_plane), (size_t)jb.nxc * nat_plane * 8,
                     cp_threads);
        }
        dn_wait += secs(t0, t1);
        dn_copy += secs(t1, clk::now());
        {
          std::lock_guard<std::mutex> lk(mu);
          if (rc && !err) err = rc;
          ++dl_done;
        }
        cv.notify_all();
      }
    });
  } else {
    for (const PipeEvent& e : plan) {
      if (e.kind != PIPE_ARRIVE) continue;
      for (Slab& s : ctx->slabs)
        if (int rc = upload_chunk(s, e)) return rc;
    }
  }
  // join the helper threads on every exit path
  struct Joiner {
    std::thread& up;
    std::thread& dn;
    std::mutex& mu;
    std::condition_variable& cv;
    bool& close;
    ~Joiner() {
      if (up.joinable()) up.join();
      {
        std::lock_guard<std::mutex> lk(mu);
        close = true;
      }
      cv.notify_all();
      if (dn.joinable()) dn.join();
    }
  } joiner{uploader, downloader, mu, cv, dl_close};

  // the wavefront on the compute streams (every slab in step); face
  // exchanges between the passes; downloads behind it
  int64_t ndl = 0;   // blocks copied back
  int64_t jdl = 0;   // download slot jobs (block x slab, staged)
  for (const PipeEvent& e : plan) {
    if (r) break;
    if (e.kind == PIPE_ARRIVE) {
      if (staged) {
        const clk::time_point t0 = clk::now();
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return arrived > e.pass || err != KGS_OK; });
        main_wait_up += secs(t0, clk::now());
        if (err) return err;
      }
      for (Slab& s : ctx->slabs) {
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamWaitEvent(s.stream, s.pipe_ev[e.pass], 0));
      }
    } else if (e.kind == PIPE_XCH) {
      if (e.pass < 0) {
        r = exchange(ctx, 0);
        if (!r) r = exchange(ctx, 1);
      } else {
        r = exchange(ctx, passes[e.pass].col);
      }
    } else if (e.kind == PIPE_PASS) {
      for (int si = 0; si < ns && !r; ++si) r = launch_range(si, passes[e.pass], e.a, e.b);
    } else {
      const int64_t k = e.pass, b0 = e.a, nxc = e.b - e.a;
      ++ndl;
      const int64_t cnt = nxc * ctx->ny * ctx->nk;
      const int blocks = (int)std::min<int64_t>((cnt + 255) / 256, (int64_t)ctx->nsm * 16);
      for (int si = 0; si < ns; ++si) {
        Slab& s = ctx->slabs[si];
        const int64_t j = staged ? jdl++ : 0;
        if (staged) {   // the download slot must have been emptied by the downloader
          const clk::time_point t0 = clk::now();
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return dl_done >= j - kDnSlots + 1 || err != KGS_OK; });
          main_wait_dn += secs(t0, clk::now());
          if (err) return err;
        }
        CK(cudaSetDevice(s.dev));
        cudaEvent_t ev = s.pipe_ev[nb + k];
        CK(cudaEventRecord(ev, s.stream));
        CK(cudaStreamWaitEvent(s.dstream, ev, 0));
        for (int f = 0; f < 4; ++f) {
          PassGeom g = make_geom(ctx, s, 1, 0, s.nx);
          g.own += f * ctx->pp;
          g.oth += f * ctx->pp;
          merge_field<<<blocks, 256, 0, s.dstream>>>(s.pipe_dn + f * C * nat_plane, g, (int)nxc,
                                                      (int)b0);
          ctx->launches++;
          double* to = staged ? dn_slot(j) + f * C * nat_plane
                              : host[f] + (s.x0 - hx0 + b0) * nat_plane;
          CK(cudaMemcpyAsync(to, s.pipe_dn + f * C * nat_plane, (size_t)nxc * nat_plane * 8,
                             cudaMemcpyDeviceToHost, s.dstream));
        }
        CK(cudaGetLastError());
        if (staged) {
          CK(cudaEventRecord(s.hslot_ev[kUpSlots + j % kDnSlots], s.dstream));
          {
            std::lock_guard<std::mutex> lk(mu);
            dl_queue.push_back({b0, nxc, j, si});
          }
          cv.notify_all();
        }
      }
    }
  }
  if (staged && !r) {   // every block copied out of its slot
    const clk::time_point t0 = clk::now();
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return dl_done >= jdl || err != KGS_OK; });
    if (dbg)
      std::fprintf(stderr, "[kgs pipe] staged call %.3f s: uploader wait %.3f copy %.3f | "
                   "downloader wait %.3f copy %.3f | main wait up %.3f dn %.3f tail %.3f\n",
                   secs(t_call, clk::now()), up_wait, up_copy, dn_wait, dn_copy, main_wait_up,
                   main_wait_dn, secs(t0, clk::now()));
    if (err) return err;
  }
  if (r) return r;
  if (ndl != nb) return fail(ctx, KGS_ECUDA, "pipeline copied back %lld of %lld blocks",
                             (long long)ndl, (long long)nb);
  for (int si = 0; si < ns; ++si) {
    Slab& s = ctx->slabs[si];
    CK(cudaSetDevice(s.dev));
    for (int64_t q = 0; q <= nrec; ++q) {
      finalize_terms<<<1, kThreads, 0, s.stream>>>(
          s.pipe_part + (q * 2 + 1) * region, (int)roff[si][q * 2 + 1],
          s.pipe_part + (q * 2) * region, (int)roff[si][q * 2], s.records + q * NTERMS);
      ctx->launches++;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(s.ev_done, s.dstream));
    CK(cudaStreamWaitEvent(s.stream, s.ev_done, 0));
    CK(cudaEventRecord(s.ev_bnd, s.stream));
  }
  CK(cudaSetDevice(s0.dev));
  for (Slab& s : ctx->slabs) CK(cudaStreamWaitEvent(s0.stream, s.ev_bnd, 0));
  CK(cudaEventRecord(s0.ev_t1, s0.stream));
  r = sync_all(ctx);
  if (r) return r;
  for (Slab& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.dstream));
    CK(cudaStreamSynchronize(s.ustream));
  }
  for (Slab& s : ctx->slabs) s.xch_pending = false;   // synchronised above
  float ms = 0.f;
  CK(cudaSetDevice(s0.dev));
  CK(cudaEventElapsedTime(&ms, s0.ev_t0, s0.ev_t1));
  ctx->last_ms = ms;
  r = read_bad(ctx, bad_out);
  if (!r) r = rank_min(ctx, bad_out);   // every rank replays to the same step
  return r;
}

}  // namespace
