/*
 * kgs_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the
 * reference's checkerboard DP-AVF2 path, used as the parity checker by
 * tests/, __graft_entry__.smoke() and as bench.py's cpu_baseline /
 * `--impl reference` leg ("port").  Never linked or called by the product
 * package (paper_2502_09537_b200/).
 *
 * It follows the reference's own structure so that its timing is a fair
 * stand-in for the reference CPU implementation:
 *   - an (M, 2d) int64 periodic neighbour table, columns (-x,+x,-y,+y,-z,+z)
 *       dpavf/grid.py:54-64 (GridSpec.neighbor_table)
 *   - red (index-sum parity 1) and black index arrays, red swept first
 *       dpavf/ordering.py:114-136 (checkerboard_schedule)
 *   - each colour phase cut into `nthreads` contiguous lanes
 *     (np.array_split) run concurrently with a barrier between phases
 *       dpavf/ordering.py:130-133, dpavf/executor.py:60-71 (PhasedExecutor)
 *   - the adjoint sweep runs phases, lanes and in-lane orders reversed
 *       dpavf/ordering.py:139-149 (reverse_schedule)
 *   - per-point arithmetic expression by expression as
 *       dpavf/kernels.py:23-54 (sweep_base) and :57-94 (sweep_adjoint)
 * Compiled with -ffp-contract=off (numba/LLVM does not contract FMAs).
 */
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* GridSpec.neighbor_table (dpavf/grid.py:54-64). */
void orc_neighbor_table(int d, int64_t N, int64_t* nbrs) {
  int64_t M = 1;
  for (int i = 0; i < d; ++i) M *= N;
  const int nn = 2 * d;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int64_t rest = i, coords[3], strides[3];
    for (int ax = d - 1; ax >= 0; --ax) {
      coords[ax] = rest % N;
      rest /= N;
    }
    int64_t s = 1;
    for (int ax = d - 1; ax >= 0; --ax) {
      strides[ax] = s;
      s *= N;
    }
    for (int ax = 0; ax < d; ++ax) {
      const int64_t cm = (coords[ax] - 1 + N) % N, cp = (coords[ax] + 1) % N;
      nbrs[i * nn + 2 * ax] = i + (cm - coords[ax]) * strides[ax];
      nbrs[i * nn + 2 * ax + 1] = i + (cp - coords[ax]) * strides[ax];
    }
  }
}

/* checkerboard_schedule colour lists (dpavf/ordering.py:125-128):
 * returns the number of red points; red[] and black[] ascending. */
int64_t orc_colour_lists(int d, int64_t N, int64_t* red, int64_t* black) {
  int64_t M = 1;
  for (int i = 0; i < d; ++i) M *= N;
  int64_t nr = 0, nb = 0;
  for (int64_t i = 0; i < M; ++i) {
    int64_t rest = i, par = 0;
    for (int ax = 0; ax < d; ++ax) {
      par += rest % N;
      rest /= N;
    }
    if (par & 1) red[nr++] = i;
    else black[nb++] = i;
  }
  return nr;
}

/* kernels.sweep_base / sweep_adjoint over one lane, in lane order
 * (reversed when `rev`).  c = kernel_args() (integrator.py:42-45). */
static void sweep_lane(double* P, double* Q, double* U, double* V,
                       const int64_t* nbrs, int nn, const int64_t* order,
                       int64_t L, int adjoint, int rev, const double* c) {
  const double alpha = c[0], beta = c[1], gcoef = c[2], c_uv = c[3],
               uv_nbr = c[4], gU = c[5], half_tau = c[6], i00 = c[7],
               i01 = c[8], i10 = c[9], i11 = c[10];
  for (int64_t t = 0; t < L; ++t) {
    const int64_t i = order[rev ? L - 1 - t : t];
    const double Pi = P[i], Qi = Q[i], Ui = U[i], Vi = V[i];
    double SP = 0.0, SQ = 0.0, SU = 0.0;
    for (int k = 0; k < nn; ++k) {
      const int64_t j = nbrs[i * nn + k];
      SP += P[j];
      SQ += Q[j];
      SU += U[j];
    }
    if (!adjoint) { /* kernels.py:43-54 */
      const double cr = gcoef * Ui - alpha;
      const double rr = -cr * Pi - Qi - beta * SP;
      const double ri = Pi - cr * Qi - beta * SQ;
      const double den = cr * cr + 1.0;
      const double Pn = (rr * cr + ri) / den;
      const double Qn = (ri * cr - rr) / den;
      P[i] = Pn;
      Q[i] = Qn;
      const double r1 = Ui + half_tau * Vi;
      const double r2 = Vi - c_uv * Ui + uv_nbr * SU + gU * (Pn * Pn + Qn * Qn);
      U[i] = i00 * r1 + i01 * r2;
      V[i] = i10 * r1 + i11 * r2;
    } else { /* kernels.py:83-94 */
      const double r1 = Ui + half_tau * Vi;
      const double r2 = Vi - c_uv * Ui + uv_nbr * SU + gU * (Pi * Pi + Qi * Qi);
      const double Un = i00 * r1 + i01 * r2;
      const double Vn = i10 * r1 + i11 * r2;
      U[i] = Un;
      V[i] = Vn;
      const double cr = gcoef * Un - alpha;
      const double rr = -cr * Pi - Qi - beta * SP;
      const double ri = Pi - cr * Qi - beta * SQ;
      const double den = cr * cr + 1.0;
      P[i] = (rr * cr + ri) / den;
      Q[i] = (ri * cr - rr) / den;
    }
  }
}

/* One colour phase: `idx` cut into `workers` np.array_split lanes, run
 * concurrently (PhasedExecutor, executor.py:60-71).  For the adjoint the
 * lanes run in reverse order with reversed in-lane order
 * (reverse_schedule, ordering.py:143-146); lanes are independent inside a
 * colour, so the result does not depend on `workers`. */
void orc_phase(double* P, double* Q, double* U, double* V,
               const int64_t* nbrs, int nn, const int64_t* idx, int64_t n,
               int adjoint, const double* c, int workers) {
  if (workers < 1) workers = 1;
  const int64_t base = n / workers, rem = n % workers;
#pragma omp parallel for schedule(static, 1) num_threads(workers)
  for (int l = 0; l < workers; ++l) {
    const int lane = adjoint ? workers - 1 - l : l;
    const int64_t start = lane * base + (lane < rem ? lane : rem);
    const int64_t len = base + (lane < rem ? 1 : 0);
    sweep_lane(P, Q, U, V, nbrs, nn, idx + start, len, adjoint, adjoint, c);
  }
}

/* nsteps of step_dpavf2 with checkerboard_schedule (integrator.py:124-129):
 * base red, base black, adjoint black, adjoint red. */
void orc_step_dpavf2(double* P, double* Q, double* U, double* V,
                     const int64_t* nbrs, int nn, const int64_t* red,
                     int64_t nred, const int64_t* black, int64_t nblack,
                     const double* c, int64_t nsteps, int workers) {
  for (int64_t s = 0; s < nsteps; ++s) {
    orc_phase(P, Q, U, V, nbrs, nn, red, nred, 0, c, workers);
    orc_phase(P, Q, U, V, nbrs, nn, black, nblack, 0, c, workers);
    orc_phase(P, Q, U, V, nbrs, nn, black, nblack, 1, c, workers);
    orc_phase(P, Q, U, V, nbrs, nn, red, nred, 1, c, workers);
  }
}

/* ------------------------------------------------------------------------
 * Table-free restatement for grids whose neighbour table does not fit in
 * host memory (1024^3: the table alone is 48 GiB, grid.py:54-64).  Same
 * per-point arithmetic as sweep_lane (kernels.py:43-54, 83-94), same
 * neighbour summation order (-x,+x,-y,+y,-z,+z; kernels.py:35-42) with the
 * periodic neighbours computed from coordinates, same colour convention
 * (red = index-sum parity 1, ordering.py:125-128) and the same phase order
 * as orc_step_dpavf2.  Inside a colour phase every update reads only
 * other-colour values, so the visiting order (here: rows in parallel) is
 * immaterial -- the bitwise-equality tests against the golden vectors pin
 * this.  The natural index is i = x*N^2 + y*N + z; axes of size 1 (the
 * missing leading axes of d = 1, 2) are skipped.
 * ---------------------------------------------------------------------- */
static void free_phase(int d, int64_t N, double* P, double* Q, double* U,
                       double* V, int colour, int adjoint, const double* c) {
  const double alpha = c[0], beta = c[1], gcoef = c[2], c_uv = c[3],
               uv_nbr = c[4], gU = c[5], half_tau = c[6], i00 = c[7],
               i01 = c[8], i10 = c[9], i11 = c[10];
  const int64_t nx = d >= 3 ? N : 1, ny = d >= 2 ? N : 1, nz = N;
  const int64_t sx = ny * nz, sy = nz;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t x = 0; x < nx; ++x) {
    for (int64_t y = 0; y < ny; ++y) {
      const int64_t xm = x == 0 ? nx - 1 : x - 1, xp = x == nx - 1 ? 0 : x + 1;
      const int64_t ym = y == 0 ? ny - 1 : y - 1, yp = y == ny - 1 ? 0 : y + 1;
      const int64_t row = x * sx + y * sy;
      const int64_t rxm = xm * sx + y * sy, rxp = xp * sx + y * sy;
      const int64_t rym = x * sx + ym * sy, ryp = x * sx + yp * sy;
      for (int64_t z = (colour + x + y) & 1; z < nz; z += 2) {
        const int64_t zm = z == 0 ? nz - 1 : z - 1, zp = z == nz - 1 ? 0 : z + 1;
        const int64_t i = row + z;
        int64_t nb[6];
        int nn = 0;
        if (nx > 1) { nb[nn++] = rxm + z; nb[nn++] = rxp + z; }
        if (ny > 1) { nb[nn++] = rym + z; nb[nn++] = ryp + z; }
        nb[nn++] = row + zm;
        nb[nn++] = row + zp;
        double SP = 0.0, SQ = 0.0, SU = 0.0;
        for (int k = 0; k < nn; ++k) {
          SP += P[nb[k]];
          SQ += Q[nb[k]];
          SU += U[nb[k]];
        }
        const double Pi = P[i], Qi = Q[i], Ui = U[i], Vi = V[i];
        if (!adjoint) { /* kernels.py:43-54 */
          const double cr = gcoef * Ui - alpha;
          const double rr = -cr * Pi - Qi - beta * SP;
          const double ri = Pi - cr * Qi - beta * SQ;
          const double den = cr * cr + 1.0;
          const double Pn = (rr * cr + ri) / den;
          const double Qn = (ri * cr - rr) / den;
          P[i] = Pn;
          Q[i] = Qn;
          const double r1 = Ui + half_tau * Vi;
          const double r2 = Vi - c_uv * Ui + uv_nbr * SU + gU * (Pn * Pn + Qn * Qn);
          U[i] = i00 * r1 + i01 * r2;
          V[i] = i10 * r1 + i11 * r2;
        } else { /* kernels.py:83-94 */
          const double r1 = Ui + half_tau * Vi;
          const double r2 = Vi - c_uv * Ui + uv_nbr * SU + gU * (Pi * Pi + Qi * Qi);
          const double Un = i00 * r1 + i01 * r2;
          const double Vn = i10 * r1 + i11 * r2;
          U[i] = Un;
          V[i] = Vn;
          const double cr = gcoef * Un - alpha;
          const double rr = -cr * Pi - Qi - beta * SP;
          const double ri = Pi - cr * Qi - beta * SQ;
          const double den = cr * cr + 1.0;
          P[i] = (rr * cr + ri) / den;
          Q[i] = (ri * cr - rr) / den;
        }
      }
    }
  }
}

/* One checkerboard sweep: base = red then black (step_base,
 * integrator.py:107-112), adjoint = black then red (step_adjoint on the
 * reversed schedule, :115-121, ordering.py:139-149). */
void orc_free_sweep(int d, int64_t N, double* P, double* Q, double* U,
                    double* V, int adjoint, const double* c) {
  free_phase(d, N, P, Q, U, V, adjoint ? 0 : 1, adjoint, c);
  free_phase(d, N, P, Q, U, V, adjoint ? 1 : 0, adjoint, c);
}

/* nsteps of step_dpavf2 (integrator.py:124-129), table-free. */
void orc_free_step_dpavf2(int d, int64_t N, double* P, double* Q, double* U,
                          double* V, const double* c, int64_t nsteps) {
  for (int64_t s = 0; s < nsteps; ++s) {
    orc_free_sweep(d, N, P, Q, U, V, 0, c);
    orc_free_sweep(d, N, P, Q, U, V, 1, c);
  }
}

/* The 8 unscaled energy sums of include/kgs_b200.h (grid.py:152-187
 * before the h-scaling), one partial per (x, y) row so the caller can sum
 * the rows exactly (math.fsum): out[row*8 + t] for
 *   t = 0..2: sum over axes of (f[+axis] - f)^2 for f = P, Q, U
 *           (np.roll(f, -1, axis) - f, grid.py:152-163)
 *   t = 3: V.V, 4: U.U, 5: (P^2 + Q^2).U, 6: P.P, 7: Q.Q. */
void orc_energy_row_terms(int d, int64_t N, const double* P, const double* Q,
                          const double* U, const double* V, double* out) {
  const int64_t nx = d >= 3 ? N : 1, ny = d >= 2 ? N : 1, nz = N;
  const int64_t sx = ny * nz, sy = nz;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t x = 0; x < nx; ++x) {
    for (int64_t y = 0; y < ny; ++y) {
      const int64_t xp = x == nx - 1 ? 0 : x + 1, yp = y == ny - 1 ? 0 : y + 1;
      const int64_t row = x * sx + y * sy;
      const double* F[3] = {P, Q, U};
      double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int64_t z = 0; z < nz; ++z) {
        const int64_t i = row + z, zp = z == nz - 1 ? 0 : z + 1;
        for (int q = 0; q < 3; ++q) {
          const double f = F[q][i];
          double a = 0.0;
          if (nx > 1) { const double e = F[q][xp * sx + y * sy + z] - f; a += e * e; }
          if (ny > 1) { const double e = F[q][x * sx + yp * sy + z] - f; a += e * e; }
          { const double e = F[q][row + zp] - f; a += e * e; }
          t[q] += a;
        }
        t[3] += V[i] * V[i];
        t[4] += U[i] * U[i];
        t[5] += (P[i] * P[i] + Q[i] * Q[i]) * U[i];
        t[6] += P[i] * P[i];
        t[7] += Q[i] * Q[i];
      }
      for (int k = 0; k < 8; ++k) out[(x * ny + y) * 8 + k] = t[k];
    }
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
