// kgs_exp_device.cuh -- EXPERIMENTAL device code, compiled only with
// -DKGS_EXPERIMENTAL (python -m paper_2502_09537_b200.build --experimental):
// the fused one-march DP-AVF2 step (step_pass).  Bitwise equal to the
// two-pass path but slower, so it is not in the default
// library.  Included from kgs_device.cuh inside namespace kgs.
#pragma once
// ---------------------------------------------------------------------------
// Fused DP-AVF2 step (d = 3): K3 (black base(n) + adjoint(n)) and K4 (red
// adjoint(n) + base(n+1), or the red adjoint tail) in ONE march that reads
// the step-n state from one buffer set and writes the result to the other
// ("ping-pong").  Every field is read once and written once per step:
// 64 B per point-step = 32 B per point-update, against 44 B for the two
// colour passes.
//
// Nothing a launch reads is written during it, so CTAs never wait on one
// another.  A unit (a TY x TK column of rows x slots, K4 planes [xs, xe))
// recomputes K3 on a one-point ring around its tile -- rows y0-1 and y0+TY,
// plus, per row, the one slot beyond the tile edge that the red
// z-neighbour on that row needs -- and on the planes xs-1 and xe, so K4 finds
// every black neighbour in its own shared memory.  Ring values and the
// extra planes are recomputed bit-identically but stored only by their
// owner (stores of K3 cover planes [wa, wb), K4 planes [xa, xb)).  Extra
// K3 work: (TY*TK + 2*TK + TY) / (TY*TK) = 1.16 at 16 x 32.
//
// Shared memory: a 4-deep ring of red planes (P, Q, U; TMA pieces: the tile,
// two halo rows above and below, two halo slots left and right over the
// tile rows and the four corner pairs at rows y0-1 / y0+TY, each at
// periodically wrapped coordinates and 128-B aligned) and a 3-deep ring of
// K3 results (black P, Q, U over rows y0-1..y0+TY and the ring column) for
// planes p-2, p-1, p.  The black own values and the red V are coalesced
// loads issued before the TMA waits.  Per plane p: K3 at p (tile, kept in
// registers, and ring), then K4 at p-1 -- its +x neighbour is this thread's
// own K3(p) result and its in-plane neighbours were completed before the
// previous barrier -- then ONE barrier and the refill of plane p+3.
// ---------------------------------------------------------------------------
struct StepGeom {
  const double* rold;   // red, step-n state (plane 0 of the set)
  const double* bold;   // black
  double* rnew;         // next state
  double* bnew;
  int64_t ps, pp;
  int rs, nx, ny, nk;
  int64_t x0;
  int wrap;             // single slab: x wraps inside the slab
  int xa, xb;           // K4 planes of this launch
  int wa, wb;           // K3 results stored for planes [wa, wb) (contains [xa, xb))
  int xc;               // K4 planes per unit
  int64_t nunits;       // ceil((xb - xa) / xc) * columns
  int dbg;              // timing experiments only (results invalid): 1 no ring K3,
                        // 2 no K4 arithmetic, 4 no K3 arithmetic
};

template <int TY, int TK>
struct StepSmem {
  static constexpr int NR = 4, NB = 3;
  static constexpr int RW = 3 * TK;              // one row: P, Q, U x TK slots
  static constexpr int CM = TY * 6;              // halo column over the tile rows: [TY][3][2]
  static constexpr int CC = 16;                  // corner pair [3][2], padded to 128 B
  static constexpr int LM = (TY + 4) * RW;       // rows y0-2 .. y0+TY+1 first
  static constexpr int RM = LM + CM;
  static constexpr int LT = RM + CM, LB = LT + CC, RT = LB + CC, RB = RT + CC;
  static constexpr int RSLOT = RB + CC;          // doubles per red slot
  static constexpr int RBYTES = ((TY + 4) * RW + 2 * CM + 4 * 6) * 8;  // TMA bytes per fill
  static constexpr int BCOL = (TY + 2) * RW;     // black slot: rows y0-1..y0+TY, then column
  static constexpr int BSLOT = BCOL + 3 * TY;
  static constexpr size_t bytes = 128 + 8 * (size_t)(NR * RSLOT + NB * BSLOT);
  static_assert(RW % 16 == 0 && CM % 16 == 0 && LM % 16 == 0 && RSLOT % 16 == 0,
                "TMA pieces must be 128-B aligned");
};

struct StepMaps {
  CUtensorMap centre;  // red (TK, 3, TY, 1)
  CUtensorMap rows2;   // red (TK, 3, 2, 1): two halo rows
  CUtensorMap col;     // red (2, 3, TY, 1): two halo slots over the tile rows
  CUtensorMap corner;  // red (2, 3, 1, 1)
};

// Neighbour sums of a colour point from shared memory, canonical order
// (-x, +x, -y, +y, -z, +z), seeded with 0.0; value triple v[0], v[fs], v[2 fs].
__device__ __forceinline__ void nb_add(double& SP, double& SQ, double& SU, const double* v,
                                       int fs) {
  SP += v[0]; SQ += v[fs]; SU += v[2 * fs];
}

// Offsets (doubles) of a point's six red neighbours inside a red slot of the
// StepSmem layout, for both z-parities: K3 at black point (r, j) of the tile
// (j in [0, TK)) or of the ring (r = -1 / TY, or j = -1 / TK).
template <int TY, int TK>
struct RedNbrs {
  int cen, cfs;          // the point's own position in a red slot (x-neighbours)
  int ym, yp, yfs;       // y-neighbours (same field stride)
  int zlo, zlofs;        // z-neighbour below (used when ob == 0) ...
  int zhi, zhifs;        // ... and above (used when ob == 1)
};

template <int TY, int TK>
__device__ __forceinline__ int red_off(int r, int j, int& fs) {
  using S = StepSmem<TY, TK>;
  if (j >= 0 && j < TK) { fs = TK; return (r + 2) * S::RW + j; }
  const bool left = j < 0;
  const int sl = left ? j + 2 : j - TK;
  fs = 2;
  if (r < 0) return (left ? S::LT : S::RT) + sl;
  if (r >= TY) return (left ? S::LB : S::RB) + sl;
  return (left ? S::LM : S::RM) + r * 6 + sl;
}

template <int TY, int TK>
__device__ __forceinline__ RedNbrs<TY, TK> red_nbrs(int r, int j) {
  RedNbrs<TY, TK> n;
  int fs;
  n.cen = red_off<TY, TK>(r, j, n.cfs);
  n.ym = red_off<TY, TK>(r - 1, j, n.yfs);
  n.yp = red_off<TY, TK>(r + 1, j, fs);
  n.zlo = red_off<TY, TK>(r, j - 1, n.zlofs);
  n.zhi = red_off<TY, TK>(r, j + 1, n.zhifs);
  return n;
}

// K3 at one black point: base(n) then adjoint(n) with the red neighbours of
// slots dm / dc / dp (planes p-1, p, p+1); ob = z-parity of the point.
template <int TY, int TK>
__device__ __forceinline__ void k3_point(const double* dm, const double* dc, const double* dp,
                                         const RedNbrs<TY, TK>& n, int ob, double& P,
                                         double& Q, double& U, double& V, const Coeffs& c) {
  double SP = 0.0, SQ = 0.0, SU = 0.0;
  nb_add(SP, SQ, SU, dm + n.cen, n.cfs);
  nb_add(SP, SQ, SU, dp + n.cen, n.cfs);
  nb_add(SP, SQ, SU, dc + n.ym, n.yfs);
  nb_add(SP, SQ, SU, dc + n.yp, n.yfs);
  if (ob) { nb_add(SP, SQ, SU, dc + n.cen, n.cfs); nb_add(SP, SQ, SU, dc + n.zhi, n.zhifs); }
  else    { nb_add(SP, SQ, SU, dc + n.zlo, n.zlofs); nb_add(SP, SQ, SU, dc + n.cen, n.cfs); }
  update_base(P, Q, U, V, SP, SQ, SU, c);
  update_adjoint(P, Q, U, V, SP, SQ, SU, c);
}

template <bool DIAG, int K4OP2, int TY, int TK, int MINB>
__global__ void __launch_bounds__(TY * TK, MINB)
step_pass(const __grid_constant__ StepMaps mr, StepGeom g, Coeffs c,
          double* __restrict__ partials, unsigned long long* __restrict__ bad, int step_no) {
  using S = StepSmem<TY, TK>;
  constexpr int NT = TY * TK, NWARP = NT / 32;
  constexpr int NRING = 2 * TK + TY;                  // ring points per plane
  constexpr int NRJ = (NRING + 31) / 32;              // ring warp jobs
  static_assert(NT % 32 == 0 && NRJ <= NWARP && TK % 32 == 0, "tile shape");
  extern __shared__ __align__(128) double smem_raw[];
  __shared__ __align__(8) unsigned long long bars[S::NR];
  double* const sR = smem_raw;                        // [NR][RSLOT]
  double* const sB = smem_raw + S::NR * S::RSLOT;     // [NB][BSLOT]

  if (threadIdx.x == 0) {
    for (int i = 0; i < S::NR; ++i) mbar_init(smem_u32(&bars[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  double acc[NTERMS];
#pragma unroll
  for (int q = 0; q < NTERMS; ++q) acc[q] = 0.0;
  unsigned badflag = 0;

  const int lk = threadIdx.x % TK, ly = threadIdx.x / TK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ring warp jobs go to warps spread over the four SM sub-partitions
  int rj = -1;
#pragma unroll
  for (int j = 0; j < NRJ; ++j)
    if (warp == (1 + 5 * j) % NWARP) rj = j;
  const int ri = rj >= 0 ? rj * 32 + lane : NRING;    // ring index, NRING = none
  const bool has_ring = ri < NRING;
  // ring point: rows -1 / TY over the tile slots, then one slot per tile row
  // (the side flips with the plane parity)
  const bool ring_col = has_ring && ri >= 2 * TK;
  const int rr = ri < TK ? -1 : (ri < 2 * TK ? TY : ri - 2 * TK);
  const int rjj = ri < TK ? ri : (ri < 2 * TK ? ri - TK : 0);

  const int cen = (ly + 2) * S::RW + lk;             // tile point in a red slot
  const int bcen = (ly + 1) * S::RW + lk;             // K4 / black results: own position
  const int bring = S::BCOL + ly * 3;                  // ring column entry of row ly

  const int nkt = g.nk / TK;
  const int64_t ncols = (int64_t)nkt * (g.ny / TY);
  const int64_t pp = g.pp, ps = g.ps;
  const bool leader = threadIdx.x == 0;
  unsigned fr = 0;                                    // red fills issued (block-uniform)

  // planes reach from xa-2 to xb+1; nx >= 4 keeps one wrap step enough
  auto wrapx = [&](int p) {
    if (g.wrap) p = p < 0 ? p + g.nx : (p >= g.nx ? p - g.nx : p);
    return p;
  };

  for (int64_t u = blockIdx.x; u < g.nunits; u += gridDim.x) {
    const int64_t col = u % ncols;
    const int xs = g.xa + (int)(u / ncols) * g.xc;
    const int xe = min(xs + g.xc, g.xb);
    const int kt = (int)(col % nkt), yt = (int)(col / nkt);
    const int y0 = yt * TY, k0 = kt * TK;
    const unsigned f0 = fr;

    // red plane r -> fill f0 + (r - xs + 2), planes xs-2 .. xe+1
    auto issue_red = [&](int r) {
      const unsigned f = f0 + (unsigned)(r - xs + 2);
      const unsigned slot = f % S::NR, bar = smem_u32(&bars[slot]);
      double* d = sR + slot * S::RSLOT;
      const int q = wrapx(r) + 1;
      KGS_ASSERT(q >= 0 && q <= g.nx + 1);
      const int y2u = (y0 == 0) ? g.ny - 2 : y0 - 2;
      const int yd = (y0 + TY == g.ny) ? 0 : y0 + TY;
      const int yu = (y0 == 0) ? g.ny - 1 : y0 - 1;
      const int kl = (k0 == 0) ? g.nk - 2 : k0 - 2;
      const int kr = (k0 + TK == g.nk) ? 0 : k0 + TK;
      mbar_expect_tx(bar, S::RBYTES);
      tma_load_4d(smem_u32(d + 2 * S::RW), &mr.centre, k0, 0, y0, q, bar);
      tma_load_4d(smem_u32(d), &mr.rows2, k0, 0, y2u, q, bar);
      tma_load_4d(smem_u32(d + (TY + 2) * S::RW), &mr.rows2, k0, 0, yd, q, bar);
      tma_load_4d(smem_u32(d + S::LM), &mr.col, kl, 0, y0, q, bar);
      tma_load_4d(smem_u32(d + S::RM), &mr.col, kr, 0, y0, q, bar);
      tma_load_4d(smem_u32(d + S::LT), &mr.corner, kl, 0, yu, q, bar);
      tma_load_4d(smem_u32(d + S::LB), &mr.corner, kl, 0, yd, q, bar);
      tma_load_4d(smem_u32(d + S::RT), &mr.corner, kr, 0, yu, q, bar);
      tma_load_4d(smem_u32(d + S::RB), &mr.corner, kr, 0, yd, q, bar);
    };
    if (leader)
      for (int r = xs - 2; r <= min(xs + 1, xe + 1); ++r) issue_red(r);
    fr = f0 + (unsigned)(xe - xs + 4);
    auto red_slot = [&](int r) { return sR + ((f0 + (unsigned)(r - xs + 2)) % S::NR) * S::RSLOT; };
    auto wait_red = [&](int r) {
      const unsigned f = f0 + (unsigned)(r - xs + 2);
      mbar_wait(smem_u32(&bars[f % S::NR]), (f / S::NR) & 1);
    };
    // black result slots rotate with the plane: slot of p is bs, of p-1 bs1, of p-2 bs2
    int bs = 0;

    const int y = y0 + ly, k = k0 + lk;
    const int64_t tile_off = (int64_t)y * g.rs + k;
    for (int p = xs - 1; p <= xe; ++p) {
      const int pw = wrapx(p);
      const int64_t xg = g.x0 + p;
      const bool store3 = (p >= xs && p < xe) || (xs == g.xa && p == xs - 1 && p >= g.wa) ||
                          (xe == g.xb && p == xe && p < g.wb);
      const int q = p - 1;                         // K4 plane
      const bool do4 = q >= xs;
      // ---- own-value loads first (their latency overlaps the TMA waits)
      KGS_ASSERT(pw >= -1 && pw <= g.nx && y < g.ny && k < g.nk);
      const double* gb = g.bold + (int64_t)pw * ps + tile_off;
      double bP = gb[0], bQ = gb[pp], bU = gb[2 * pp], bV = gb[3 * pp];
      // ring column side: the red z-neighbour's on row rr of plane p
      const int side = ring_col ? (int)((xg + y0 + rr + 1) & 1) : 0;
      const int rjp = ring_col ? (side ? TK : -1) : rjj;   // ring point slot (tile-relative)
      double cP = 0, cQ = 0, cU = 0, cV = 0;
      if (has_ring) {
        int ry = y0 + rr, rk = k0 + rjp;
        ry = ry < 0 ? ry + g.ny : (ry >= g.ny ? ry - g.ny : ry);
        rk = rk < 0 ? rk + g.nk : (rk >= g.nk ? rk - g.nk : rk);
        KGS_ASSERT(ry >= 0 && ry < g.ny && rk >= 0 && rk < g.nk);
        const double* gr = g.bold + (int64_t)pw * ps + (int64_t)ry * g.rs + rk;
        cP = gr[0]; cQ = gr[pp]; cU = gr[2 * pp]; cV = gr[3 * pp];
      }
      const int qw = do4 ? wrapx(q) : 0;
      double rV = 0.0;
      if (do4) rV = g.rold[(int64_t)qw * ps + 3 * pp + tile_off];

      wait_red(p - 1); wait_red(p); wait_red(p + 1);
      const double* dm = red_slot(p - 1);
      const double* dc = red_slot(p);
      const double* dp = red_slot(p + 1);
      const int bs1 = bs == 0 ? 2 : bs - 1, bs2 = bs1 == 0 ? 2 : bs1 - 1;
      double* bn = sB + bs * S::BSLOT;

      // ---- K3 at the tile point of plane p (kept in registers for K4's +x)
      const int ob = (int)((xg + y) & 1);
      {
        RedNbrs<TY, TK> nt;
        nt.cen = cen; nt.cfs = TK;
        nt.ym = cen - S::RW; nt.yp = cen + S::RW; nt.yfs = TK;
        nt.zlo = (lk == 0) ? S::LM + ly * 6 + 1 : cen - 1;
        nt.zlofs = (lk == 0) ? 2 : TK;
        nt.zhi = (lk == TK - 1) ? S::RM + ly * 6 : cen + 1;
        nt.zhifs = (lk == TK - 1) ? 2 : TK;
        if (!(g.dbg & 4)) k3_point<TY, TK>(dm, dc, dp, nt, ob, bP, bQ, bU, bV, c);
      }
      bn[bcen] = bP; bn[bcen + TK] = bQ; bn[bcen + 2 * TK] = bU;
      if (store3) {
        badflag |= non_finite(bP) | non_finite(bQ) | non_finite(bU) | non_finite(bV);
        if (DIAG) {
          const double pq = bP * bP + bQ * bQ;
          acc[3] += bV * bV; acc[4] += bU * bU; acc[5] += pq * bU;
          acc[6] += bP * bP; acc[7] += bQ * bQ;
        }
        KGS_ASSERT(pw >= 0 && pw < g.nx);
        double* w = g.bnew + (int64_t)pw * ps + tile_off;
        w[0] = bP; w[pp] = bQ; w[2 * pp] = bU; w[3 * pp] = bV;
      }
      // ---- K3 at the ring point of plane p (read by K4(p) next iteration)
      if (has_ring && !(g.dbg & 1)) {
        const int rob = (int)((xg + y0 + rr) & 1);
        k3_point<TY, TK>(dm, dc, dp, red_nbrs<TY, TK>(rr, rjp), rob, cP, cQ, cU, cV, c);
        if (!ring_col) {
          double* o = bn + (rr + 1) * S::RW + rjj;
          o[0] = cP; o[TK] = cQ; o[2 * TK] = cU;
        } else {
          double* o = bn + S::BCOL + rr * 3;
          o[0] = cP; o[1] = cQ; o[2] = cU;
        }
      }

      // ---- K4 at the red tile point of plane q = p - 1: black +x from the
      // registers above, -x from this thread's own entry of slot q-1, and the
      // in-plane neighbours from slot q (complete since the last barrier)
      if (do4) {
        const double* sq = red_slot(q) + cen;
        double P = sq[0], Q = sq[TK], U = sq[2 * TK], V = rV;
        const double* bm = sB + bs2 * S::BSLOT + bcen;
        const double* bc = sB + bs1 * S::BSLOT;
        const int orr = (int)((g.x0 + q + y + 1) & 1);
        const double* zlo = (lk == 0) ? bc + bring : bc + bcen - 1;
        const int zlofs = (lk == 0) ? 1 : TK;
        const double* zhi = (lk == TK - 1) ? bc + bring : bc + bcen + 1;
        const int zhifs = (lk == TK - 1) ? 1 : TK;
        const double* z1 = orr ? bc + bcen : zlo;
        const int z1fs = orr ? TK : zlofs;
        const double* z2 = orr ? zhi : bc + bcen;
        const int z2fs = orr ? zhifs : TK;
        double SP = 0.0, SQ = 0.0, SU = 0.0;
        nb_add(SP, SQ, SU, bm, TK);
        SP += bP; SQ += bQ; SU += bU;
        nb_add(SP, SQ, SU, bc + bcen - S::RW, TK);
        nb_add(SP, SQ, SU, bc + bcen + S::RW, TK);
        nb_add(SP, SQ, SU, z1, z1fs);
        nb_add(SP, SQ, SU, z2, z2fs);
        if (!(g.dbg & 2)) update_adjoint(P, Q, U, V, SP, SQ, SU, c);
        else P += SP + SQ + SU;
        badflag |= non_finite(P) | non_finite(Q) | non_finite(U) | non_finite(V);
        if (DIAG) {
          const double pq = P * P + Q * Q;
          acc[3] += V * V; acc[4] += U * U; acc[5] += pq * U;
          acc[6] += P * P; acc[7] += Q * Q;
          auto edge = [&](double a, double b, double e) {
            const double ep = a - P, eq = b - Q, eu = e - U;
            acc[0] += ep * ep; acc[1] += eq * eq; acc[2] += eu * eu;
          };
          edge(bm[0], bm[TK], bm[2 * TK]);
          edge(bP, bQ, bU);
          const double* v = bc + bcen - S::RW;
          edge(v[0], v[TK], v[2 * TK]);
          v = bc + bcen + S::RW;
          edge(v[0], v[TK], v[2 * TK]);
          edge(z1[0], z1[z1fs], z1[2 * z1fs]);
          edge(z2[0], z2[z2fs], z2[2 * z2fs]);
        }
        if (!(g.dbg & 2)) apply_op<K4OP2>(P, Q, U, V, SP, SQ, SU, c);
        KGS_ASSERT(qw >= 0 && qw < g.nx && q >= g.xa && q < g.xb);
        double* w = g.rnew + (int64_t)qw * ps + tile_off;
        w[0] = P; w[pp] = Q; w[2 * pp] = U; w[3 * pp] = V;
      }
      __syncthreads();   // black slot p complete; red slot p-1 and black slot p-2 free
      if (leader && p + 3 <= xe + 1) issue_red(p + 3);
      bs = bs == 2 ? 0 : bs + 1;
    }
  }

  if (__syncthreads_or(badflag != 0) && threadIdx.x == 0)
    atomicMin(bad, (unsigned long long)step_no);
  if (DIAG) block_reduce_store(acc, partials + (int64_t)blockIdx.x * NTERMS);
}

// ---------------------------------------------------------------------------
// Fused step, second form (step2_pass, knob fused_step = 2).  Same ping-pong
// sets and ring recomputation as step_pass, but K4 runs TWO planes behind K3
// (K3 at plane p, K4 at p-2): every black value K4 needs -- planes p-3, p-2,
// p-1 and the ring -- was finished in earlier iterations, so the K3 chain at
// p and the K4 chain at p-2 of a thread are independent.  They are written
// stage by stage (K3 base-psi with K4 adjoint-uv, K3 base-uv with K4
// adjoint-psi, ...), each stage holding exactly one exact-division fallback
// branch, so the scheduler interleaves the two chains (the two-rows-per-
// thread ILP of the two-pass march).  Rings: red 5 slots (planes p-2..p+2),
// black results 4 slots (p-3..p).
// ---------------------------------------------------------------------------
template <int TY, int TK, int NR_, int NB_>
struct Step2Smem {
  using B = StepSmem<TY, TK>;
  static constexpr int NR = NR_, NB = NB_;
  static constexpr int RW = B::RW, LM = B::LM, RM = B::RM, LT = B::LT, LB = B::LB, RT = B::RT,
                       RB = B::RB, RSLOT = B::RSLOT, RBYTES = B::RBYTES, BCOL = B::BCOL,
                       BSLOT = B::BSLOT;
  static constexpr size_t bytes = 128 + 8 * (size_t)(NR * RSLOT + NB * BSLOT);
};

template <bool DIAG, int K4OP2, int TY, int TK, int MINB>
__global__ void __launch_bounds__(TY * TK, MINB)
step2_pass(const __grid_constant__ StepMaps mr, StepGeom g, Coeffs c,
           double* __restrict__ partials, unsigned long long* __restrict__ bad, int step_no) {
  using S = Step2Smem<TY, TK, 5, 4>;
  constexpr int NT = TY * TK, NWARP = NT / 32;
  constexpr int NRING = 2 * TK + TY;                  // ring points per plane
  constexpr int NRJ = (NRING + 31) / 32;              // ring warp jobs
  static_assert(NT % 32 == 0 && NRJ <= NWARP && TK % 32 == 0, "tile shape");
  extern __shared__ __align__(128) double smem_raw[];
  __shared__ __align__(8) unsigned long long bars[S::NR];
  double* const sR = smem_raw;                        // [NR][RSLOT]
  double* const sB = smem_raw + S::NR * S::RSLOT;     // [NB][BSLOT]

  if (threadIdx.x == 0) {
    for (int i = 0; i < S::NR; ++i) mbar_init(smem_u32(&bars[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  double acc[NTERMS];
#pragma unroll
  for (int q = 0; q < NTERMS; ++q) acc[q] = 0.0;
  unsigned badflag = 0;

  const int lk = threadIdx.x % TK, ly = threadIdx.x / TK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int rj = -1;
#pragma unroll
  for (int j = 0; j < NRJ; ++j)
    if (warp == (1 + 5 * j) % NWARP) rj = j;
  const int ri = rj >= 0 ? rj * 32 + lane : NRING;
  const bool has_ring = ri < NRING;
  const bool ring_col = has_ring && ri >= 2 * TK;
  const int rr = ri < TK ? -1 : (ri < 2 * TK ? TY : ri - 2 * TK);
  const int rjj = ri < TK ? ri : (ri < 2 * TK ? ri - TK : 0);

  const int cen = (ly + 2) * S::RW + lk;             // tile point in a red slot
  const int bcen = (ly + 1) * S::RW + lk;             // tile point in a black slot
  const int bring = S::BCOL + ly * 3;

  const int nkt = g.nk / TK;
  const int64_t ncols = (int64_t)nkt * (g.ny / TY);
  const int64_t pp = g.pp, ps = g.ps;
  const bool leader = threadIdx.x == 0;
  unsigned fr = 0;

  auto wrapx = [&](int p) {
    if (g.wrap) p = p < 0 ? p + g.nx : (p >= g.nx ? p - g.nx : p);
    return p;
  };

  for (int64_t u = blockIdx.x; u < g.nunits; u += gridDim.x) {
    const int64_t col = u % ncols;
    const int xs = g.xa + (int)(u / ncols) * g.xc;
    const int xe = min(xs + g.xc, g.xb);
    const int kt = (int)(col % nkt), yt = (int)(col / nkt);
    const int y0 = yt * TY, k0 = kt * TK;
    const unsigned f0 = fr;

    // red plane r -> fill f0 + (r - xs + 2), planes xs-2 .. xe+1
    auto issue_red = [&](int r) {
      const unsigned f = f0 + (unsigned)(r - xs + 2);
      const unsigned slot = f % S::NR, bar = smem_u32(&bars[slot]);
      double* d = sR + slot * S::RSLOT;
      const int q = wrapx(r) + 1;
      KGS_ASSERT(q >= 0 && q <= g.nx + 1);
      const int y2u = (y0 == 0) ? g.ny - 2 : y0 - 2;
      const int yd = (y0 + TY == g.ny) ? 0 : y0 + TY;
      const int yu = (y0 == 0) ? g.ny - 1 : y0 - 1;
      const int kl = (k0 == 0) ? g.nk - 2 : k0 - 2;
      const int kr = (k0 + TK == g.nk) ? 0 : k0 + TK;
      mbar_expect_tx(bar, S::RBYTES);
      tma_load_4d(smem_u32(d + 2 * S::RW), &mr.centre, k0, 0, y0, q, bar);
      tma_load_4d(smem_u32(d), &mr.rows2, k0, 0, y2u, q, bar);
      tma_load_4d(smem_u32(d + (TY + 2) * S::RW), &mr.rows2, k0, 0, yd, q, bar);
      tma_load_4d(smem_u32(d + S::LM), &mr.col, kl, 0, y0, q, bar);
      tma_load_4d(smem_u32(d + S::RM), &mr.col, kr, 0, y0, q, bar);
      tma_load_4d(smem_u32(d + S::LT), &mr.corner, kl, 0, yu, q, bar);
      tma_load_4d(smem_u32(d + S::LB), &mr.corner, kl, 0, yd, q, bar);
      tma_load_4d(smem_u32(d + S::RT), &mr.corner, kr, 0, yu, q, bar);
      tma_load_4d(smem_u32(d + S::RB), &mr.corner, kr, 0, yd, q, bar);
    };
    if (leader)   // planes xs-2 .. xs+1; then after iteration p the slot of p-2 takes p+3
      for (int r = xs - 2; r <= min(xs + 1, xe + 1); ++r) issue_red(r);
    fr = f0 + (unsigned)(xe - xs + 4);
    auto red_slot = [&](int r) { return sR + ((f0 + (unsigned)(r - xs + 2)) % S::NR) * S::RSLOT; };
    auto wait_red = [&](int r) {
      const unsigned f = f0 + (unsigned)(r - xs + 2);
      mbar_wait_wd(smem_u32(&bars[f % S::NR]), (f / S::NR) & 1);   // traps, never hangs
    };
    auto black_slot = [&](int p) { return sB + ((unsigned)(p - xs + 1) % S::NB) * S::BSLOT; };

    const int y = y0 + ly, k = k0 + lk;
    const int64_t tile_off = (int64_t)y * g.rs + k;
    for (int p = xs - 1; p <= xe + 1; ++p) {
      const bool do3 = p <= xe;
      const int q = p - 2;                         // K4 plane
      const bool do4 = q >= xs && q < xe;
      const int pw = do3 ? wrapx(p) : 0;
      const int qw = do4 ? wrapx(q) : 0;
      const int64_t xg = g.x0 + p;
      const bool store3 = do3 && ((p >= xs && p < xe) || (xs == g.xa && p == xs - 1 && p >= g.wa) ||
                                  (xe == g.xb && p == xe && p < g.wb));
      // ---- own-value loads first (their latency overlaps the TMA waits)
      double bP = 0, bQ = 0, bU = 0, bV = 0, cP = 0, cQ = 0, cU = 0, cV = 0, rV = 0;
      int rjp = 0;
      if (do3) {
        KGS_ASSERT(pw >= -1 && pw <= g.nx && y < g.ny && k < g.nk);
        const double* gb = g.bold + (int64_t)pw * ps + tile_off;
        bP = gb[0]; bQ = gb[pp]; bU = gb[2 * pp]; bV = gb[3 * pp];
        const int side = ring_col ? (int)((xg + y0 + rr + 1) & 1) : 0;
        rjp = ring_col ? (side ? TK : -1) : rjj;
        if (has_ring) {
          int ry = y0 + rr, rk = k0 + rjp;
          ry = ry < 0 ? ry + g.ny : (ry >= g.ny ? ry - g.ny : ry);
          rk = rk < 0 ? rk + g.nk : (rk >= g.nk ? rk - g.nk : rk);
          KGS_ASSERT(ry >= 0 && ry < g.ny && rk >= 0 && rk < g.nk);
          const double* gr = g.bold + (int64_t)pw * ps + (int64_t)ry * g.rs + rk;
          cP = gr[0]; cQ = gr[pp]; cU = gr[2 * pp]; cV = gr[3 * pp];
        }
      }
      if (do4) rV = g.rold[(int64_t)qw * ps + 3 * pp + tile_off];
      if (do3) { wait_red(p - 1); wait_red(p); wait_red(p + 1); }

      // ---- neighbour sums: K3 at the black tile point of plane p, K4 at the
      // red tile point of plane q (black results of planes q-1, q, q+1)
      double P3[1] = {bP}, Q3[1] = {bQ}, U3[1] = {bU}, V3[1] = {bV};
      double S3P[1] = {0.0}, S3Q[1] = {0.0}, S3U[1] = {0.0};
      const int ob = (int)((xg + y) & 1);
      if (do3) {
        const double* dm = red_slot(p - 1);
        const double* dc = red_slot(p);
        const double* dp = red_slot(p + 1);
        const int zlo = (lk == 0) ? S::LM + ly * 6 + 1 : cen - 1;
        const int zlofs = (lk == 0) ? 2 : TK;
        const int zhi = (lk == TK - 1) ? S::RM + ly * 6 : cen + 1;
        const int zhifs = (lk == TK - 1) ? 2 : TK;
        nb_add(S3P[0], S3Q[0], S3U[0], dm + cen, TK);
        nb_add(S3P[0], S3Q[0], S3U[0], dp + cen, TK);
        nb_add(S3P[0], S3Q[0], S3U[0], dc + cen - S::RW, TK);
        nb_add(S3P[0], S3Q[0], S3U[0], dc + cen + S::RW, TK);
        if (ob) { nb_add(S3P[0], S3Q[0], S3U[0], dc + cen, TK);
                  nb_add(S3P[0], S3Q[0], S3U[0], dc + zhi, zhifs); }
        else    { nb_add(S3P[0], S3Q[0], S3U[0], dc + zlo, zlofs);
                  nb_add(S3P[0], S3Q[0], S3U[0], dc + cen, TK); }
      }
      double P4[1] = {0.0}, Q4[1] = {0.0}, U4[1] = {0.0}, V4[1] = {rV};
      double S4P[1] = {0.0}, S4Q[1] = {0.0}, S4U[1] = {0.0};
      const double *bm = nullptr, *bpx = nullptr, *z1 = nullptr, *z2 = nullptr, *bc = nullptr;
      int z1fs = TK, z2fs = TK;
      if (do4) {
        const double* sq = red_slot(q) + cen;
        P4[0] = sq[0]; Q4[0] = sq[TK]; U4[0] = sq[2 * TK];
        bm = black_slot(q - 1) + bcen;
        bpx = black_slot(q + 1) + bcen;
        bc = black_slot(q);
        const int orr = (int)((g.x0 + q + y + 1) & 1);
        const double* zlo = (lk == 0) ? bc + bring : bc + bcen - 1;
        const int zlofs = (lk == 0) ? 1 : TK;
        const double* zhi = (lk == TK - 1) ? bc + bring : bc + bcen + 1;
        const int zhifs = (lk == TK - 1) ? 1 : TK;
        z1 = orr ? bc + bcen : zlo;
        z1fs = orr ? TK : zlofs;
        z2 = orr ? zhi : bc + bcen;
        z2fs = orr ? zhifs : TK;
        nb_add(S4P[0], S4Q[0], S4U[0], bm, TK);
        nb_add(S4P[0], S4Q[0], S4U[0], bpx, TK);
        nb_add(S4P[0], S4Q[0], S4U[0], bc + bcen - S::RW, TK);
        nb_add(S4P[0], S4Q[0], S4U[0], bc + bcen + S::RW, TK);
        nb_add(S4P[0], S4Q[0], S4U[0], z1, z1fs);
        nb_add(S4P[0], S4Q[0], S4U[0], z2, z2fs);
      }

      // ---- the two chains, stage by stage (one division branch per stage):
      // K3 = base (psi, uv) then adjoint (uv, psi); K4 = adjoint (uv, psi)
      // then K4OP2 (base: psi, uv)
      if (do4) uv_solve_n<1>(U4, V4, P4, Q4, S4U, c);
      if (do3) psi_solve_n<1>(P3, Q3, U3, S3P, S3Q, c);
      if (do3) uv_solve_n<1>(U3, V3, P3, Q3, S3U, c);
      if (do4) psi_solve_n<1>(P4, Q4, U4, S4P, S4Q, c);
      if (do4) {   // the step-n red state: finiteness and record terms
        badflag |= non_finite(P4[0]) | non_finite(Q4[0]) | non_finite(U4[0]) | non_finite(V4[0]);
        if (DIAG) {
          const double P = P4[0], Q = Q4[0], U = U4[0], V = V4[0];
          const double pq = P * P + Q * Q;
          acc[3] += V * V; acc[4] += U * U; acc[5] += pq * U;
          acc[6] += P * P; acc[7] += Q * Q;
          auto edge = [&](const double* v, int fs) {
            const double ep = v[0] - P, eq = v[fs] - Q, eu = v[2 * fs] - U;
            acc[0] += ep * ep; acc[1] += eq * eq; acc[2] += eu * eu;
          };
          edge(bm, TK); edge(bpx, TK);
          edge(bc + bcen - S::RW, TK); edge(bc + bcen + S::RW, TK);
          edge(z1, z1fs); edge(z2, z2fs);
        }
      }
      if (do3) uv_solve_n<1>(U3, V3, P3, Q3, S3U, c);
      if (K4OP2 == OP_BASE && do4) psi_solve_n<1>(P4, Q4, U4, S4P, S4Q, c);
      if (K4OP2 == OP_BASE && do4) uv_solve_n<1>(U4, V4, P4, Q4, S4U, c);
      if (do3) psi_solve_n<1>(P3, Q3, U3, S3P, S3Q, c);

      if (do3) {
        double* bn = black_slot(p);
        bn[bcen] = P3[0]; bn[bcen + TK] = Q3[0]; bn[bcen + 2 * TK] = U3[0];
        if (store3) {
          badflag |= non_finite(P3[0]) | non_finite(Q3[0]) | non_finite(U3[0]) | non_finite(V3[0]);
          if (DIAG) {
            const double pq = P3[0] * P3[0] + Q3[0] * Q3[0];
            acc[3] += V3[0] * V3[0]; acc[4] += U3[0] * U3[0]; acc[5] += pq * U3[0];
            acc[6] += P3[0] * P3[0]; acc[7] += Q3[0] * Q3[0];
          }
          KGS_ASSERT(pw >= 0 && pw < g.nx);
          double* w = g.bnew + (int64_t)pw * ps + tile_off;
          w[0] = P3[0]; w[pp] = Q3[0]; w[2 * pp] = U3[0]; w[3 * pp] = V3[0];
        }
        // ---- K3 at the ring point of plane p (read by K4 at q = p)
        if (has_ring && !(g.dbg & 1)) {
          const int rob = (int)((xg + y0 + rr) & 1);
          k3_point<TY, TK>(red_slot(p - 1), red_slot(p), red_slot(p + 1),
                           red_nbrs<TY, TK>(rr, rjp), rob, cP, cQ, cU, cV, c);
          if (!ring_col) {
            double* o = bn + (rr + 1) * S::RW + rjj;
            o[0] = cP; o[TK] = cQ; o[2 * TK] = cU;
          } else {
            double* o = bn + S::BCOL + rr * 3;
            o[0] = cP; o[1] = cQ; o[2] = cU;
          }
        }
      }
      if (do4) {
        KGS_ASSERT(qw >= 0 && qw < g.nx && q >= g.xa && q < g.xb);
        double* w = g.rnew + (int64_t)qw * ps + tile_off;
        w[0] = P4[0]; w[pp] = Q4[0]; w[2 * pp] = U4[0]; w[3 * pp] = V4[0];
      }
      __syncthreads();   // black slot p complete; red slot p-2 and black slot p-3 free
      if (leader && p + 3 <= xe + 1) issue_red(p + 3);
    }
  }

  if (__syncthreads_or(badflag != 0) && threadIdx.x == 0)
    atomicMin(bad, (unsigned long long)step_no);
  if (DIAG) block_reduce_store(acc, partials + (int64_t)blockIdx.x * NTERMS);
}
