// kgs_passes.cuh -- colour passes over all slabs: halo exchange (NCCL / copies / fused stores), interior/boundary split, timing, records, allocation.
// Part of the single translation unit kgs_host.cu (included in order).
#pragma once

namespace {

// ---- halo exchange of colour `col` faces (P, Q, U of planes 0 and nx-1) --
// The three fields of a plane are contiguous ([P|Q|U|V] per plane), so a
// face is ONE contiguous run of 3*pp doubles.
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

// Ranks of a torchrun job agree on a value: the minimum over ranks (an NCCL
// all-reduce every rank must reach at the same point).  Otherwise a no-op --
// except for a self-exchanging rank (KGS_SELF_EXCHANGE), which runs the
// 1-rank all-reduce so that this path executes on one GPU too.
int rank_min(kgs_ctx* ctx, unsigned long long* v) {
  if (!(ctx->dist && (ctx->nranks > 1 || ctx->self_xch))) return KGS_OK;
  Slab& s = ctx->slabs[0];
  CK(cudaSetDevice(s.dev));
  if (!ctx->dword) CK(cudaMalloc(&ctx->dword, sizeof(unsigned long long)));
  CK(cudaMemcpyAsync(ctx->dword, v, sizeof *v, cudaMemcpyHostToDevice, s.cstream));
  NK(g_nccl.AllReduce(ctx->dword, ctx->dword, 1, ncclUint64, ncclMin, ctx->comm, s.cstream));
  CK(cudaMemcpyAsync(v, ctx->dword, sizeof *v, cudaMemcpyDeviceToHost, s.cstream));
  CK(cudaStreamSynchronize(s.cstream));
  return KGS_OK;
}

int finalize_record(kgs_ctx* ctx, int64_t slot, bool both);

int sync_all(kgs_ctx* ctx) {
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.stream));
    CK(cudaStreamSynchronize(s.cstream));
    CK(cudaStreamSynchronize(s.fstream));
    s.fin_busy[0] = s.fin_busy[1] = false;
  }
  return KGS_OK;
}

// ---- program executor (kgs_program.cuh) --------------------------------
// Every slab executes the program in order on its compute stream; halo
// exchanges run on its comm stream.  Ordering is by stream events only:
//  * PG_XCH records ev_bnd (the faces are written) and starts the exchange
//    (NCCL send/recv or peer copies) on the comm stream, completing ev_xch;
//  * PG_WAIT_XCH makes the compute stream wait for ev_xch -- placed after
//    a pass's interior launch, so the interior overlaps the transfer, and
//    before the boundary launches that read the ghosts.
// Fused halo exchange (ctx->mirror: single process, peer-accessible
// neighbours): the boundary launches of slab i also store their new faces
// into the neighbours' ghost planes (peer pointers), so the PG_XCH that
// follows is a no-op.  Then PG_WAIT_XCH of pass k also waits for both
// neighbours' boundary launches of pass k-1 (ev_face): that is when they
// finished writing i's ghosts (RAW) and finished reading their own ghosts
// that i is about to overwrite (WAR); pending copy exchanges into either
// side (after uploads) are waited for as well.
int run_program(kgs_ctx* ctx, const Program& prog, const Coeffs& c) {
  const bool split = needs_exchange(ctx);
  const bool mirror = split && ctx->mirror && ctx->tune_mirror;
  const int ns = (int)ctx->slabs.size();
  int64_t k = 0;            // number of the current pass (fused halo stores)
  bool in_pass = false, writes = false, timing = false;
  int pcol = 0;
  for (const ProgOp& o : prog) {
    switch (o.kind) {
      case PG_PASS_BEGIN: {
        in_pass = true;
        pcol = o.col;
        writes = o.op1 != OP_NONE || o.op2 != OP_NONE;
        k = ctx->pass_no;
        if (split) ctx->pass_no++;
        int64_t pts = 0;
        for (auto& s : ctx->slabs) {
          if (o.diag) {
            s.npart[o.col] = 0;
            if (s.fin_busy[s.pset]) {   // a record reduction still reads this set
              CK(cudaSetDevice(s.dev));
              CK(cudaStreamWaitEvent(s.stream, s.ev_fin[s.pset], 0));
              s.fin_busy[s.pset] = false;
            }
          }
          pts += (int64_t)s.nx * ctx->ny * ctx->nk;
        }
        timing = o.xa && ctx->pass_timing;
        if (o.xa) ctx->timed_pts = pts;
        if (timing) {   // event pair on slab 0's stream around the fused pass
          Slab& s0 = ctx->slabs[0];
          CK(cudaSetDevice(s0.dev));
          if (ctx->pass_ev_used + 2 > ctx->pass_ev.size())
            for (int i = 0; i < 64; ++i) {
              cudaEvent_t e;
              CK(cudaEventCreate(&e));
              ctx->pass_ev.push_back(e);
            }
          CK(cudaEventRecord(ctx->pass_ev[ctx->pass_ev_used++], s0.stream));
        }
        break;
      }
      case PG_LAUNCH:
        for (int i = 0; i < ns; ++i) {
          Slab& s = ctx->slabs[i];
          cudaError_t e = cudaSetDevice(s.dev);
          if (e != cudaSuccess)
            return fail(ctx, KGS_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
          const int xb = std::min(o.xb, s.nx);
          // our plane 0 is lo's ghost plane lo.nx; our plane nx-1 is hi's ghost -1
          double* mlo = nullptr;
          double* mhi = nullptr;
          if (mirror && writes) {
            Slab& lo = ctx->slabs[(i - 1 + ns) % ns];
            Slab& hi = ctx->slabs[(i + 1) % ns];
            if (o.xa == 0) mlo = lo.plane0[o.col] + (int64_t)lo.nx * ctx->ps;
            if (xb == s.nx) mhi = hi.plane0[o.col] - ctx->ps;
          }
          int r = launch_pass(ctx, s, o.col, o.op1, o.op2, o.diag != 0, o.check != 0, c, o.step,
                              o.xa, xb, nullptr, mlo, mhi);
          if (r) return r;
        }
        break;
      case PG_WAIT_XCH:
        for (int i = 0; i < ns; ++i) {
          Slab& s = ctx->slabs[i];
          CK(cudaSetDevice(s.dev));
          if (s.xch_pending) {
            CK(cudaStreamWaitEvent(s.stream, s.ev_xch, 0));
            s.xch_pending = false;
          }
          if (mirror && in_pass) {
            Slab& lo = ctx->slabs[(i - 1 + ns) % ns];
            Slab& hi = ctx->slabs[(i + 1) % ns];
            CK(cudaStreamWaitEvent(s.stream, lo.ev_xch, 0));
            CK(cudaStreamWaitEvent(s.stream, hi.ev_xch, 0));
            if (k > 0) {
              CK(cudaStreamWaitEvent(s.stream, lo.ev_face[(k - 1) & 1], 0));
              CK(cudaStreamWaitEvent(s.stream, hi.ev_face[(k - 1) & 1], 0));
            }
          }
        }
        break;
      case PG_PASS_END:
        if (mirror)
          for (auto& s : ctx->slabs) {
            CK(cudaSetDevice(s.dev));
            CK(cudaEventRecord(s.ev_face[k & 1], s.stream));
          }
        if (mirror && writes) ctx->mirrored[pcol] = true;
        if (timing) {
          Slab& s0 = ctx->slabs[0];
          CK(cudaSetDevice(s0.dev));
          CK(cudaEventRecord(ctx->pass_ev[ctx->pass_ev_used++], s0.stream));
        }
        in_pass = timing = false;
        break;
      case PG_XCH: {
        int r = exchange(ctx, o.col);
        if (r) return r;
        break;
      }
      case PG_RECORD: {
        int r = finalize_record(ctx, o.step, o.xa != 0);
        if (r) return r;
        break;
      }
      case PG_DEFER:
        ctx->pending = true;
        ctx->pend_c = c;
        break;
      default:
        return fail(ctx, KGS_EINVAL, "bad program op %d", o.kind);
    }
  }
  return KGS_OK;
}

// One colour pass over every slab (no exchange after it).
int all_passes(kgs_ctx* ctx, int col, int op1, int op2, bool diag, bool check,
               const Coeffs& c, int step_no) {
  const Program p = pass_program(ctx->slabs[0].nx, needs_exchange(ctx), col, op1, op2, diag,
                                 check, step_no, false);
  return run_program(ctx, p, c);
}

#ifdef KGS_EXPERIMENTAL
// Run `launch` bracketed by an event pair on slab 0's stream when timing
// (the experimental fused step).
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
#endif

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

// Reduce the current partial set into record `slot` on the slab's record
// stream, after the passes that wrote it, and switch the passes to the other
// set: the next steps' passes do not wait for the reduction (the set is
// only written again two records later, after waiting for ev_fin).
int finalize_record(kgs_ctx* ctx, int64_t slot, bool both) {
  for (auto& s : ctx->slabs) {
    CK(cudaSetDevice(s.dev));
    CK(cudaEventRecord(s.ev_diag, s.stream));
    CK(cudaStreamWaitEvent(s.fstream, s.ev_diag, 0));
    finalize_terms<<<1, kThreads, 0, s.fstream>>>(
        (const double*)s.partials[1], s.npart[1], (const double*)(both ? s.partials[0] : nullptr),
        both ? s.npart[0] : 0, s.records + slot * NTERMS);
    CK(cudaGetLastError());
    CK(cudaEventRecord(s.ev_fin[s.pset], s.fstream));
    s.fin_busy[s.pset] = true;
    std::swap(s.partials[0], s.partials_alt[0]);
    std::swap(s.partials[1], s.partials_alt[1]);
    s.pset ^= 1;
    ctx->launches++;
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
    CK(cudaMalloc(&s.partials_alt[c], (size_t)4 * ctx->grid_cap * NTERMS * sizeof(double)));
  }
  if (ctx->d == 3) {
    int r = make_tensor_maps(ctx, s);
    if (r) return r;
  }
  CK(cudaMalloc(&s.bad, sizeof(unsigned long long)));
  CK(cudaMemset(s.bad, 0xff, sizeof(unsigned long long)));
  CK(cudaMalloc(&s.wctr, sizeof(unsigned long long)));
  CK(cudaMemset(s.wctr, 0, sizeof(unsigned long long)));
  s.wbase = 0;

  // staging: up to 256 MiB of natural-layout planes of one field
  const size_t nat_plane = (size_t)ctx->ny * ctx->nz * sizeof(double);
  s.stage_planes = (int)std::max<size_t>(1, std::min<size_t>(s.nx, (256u << 20) / nat_plane));
  CK(cudaMalloc(&s.stage, s.stage_planes * nat_plane));
  CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s.cstream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s.fstream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&s.ev_fin[i], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_diag, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_bnd, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_xch, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i)
    CK(cudaEventCreateWithFlags(&s.ev_face[i], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming));
  CK(cudaEventCreate(&s.ev_t0));
  CK(cudaEventCreate(&s.ev_t1));
  // the zero-fills above run on the legacy default stream, which the
  // non-blocking slab streams do not wait for: finish them before any use
  CK(cudaDeviceSynchronize());
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
