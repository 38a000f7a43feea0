// kgs_program.cuh -- the pass program of a call: a pure host list of what
// every slab (or rank) does, in order -- colour-pass launches over plane
// ranges, halo exchanges, waits for them, energy records, the deferred
// tail.  kgs_passes.cuh executes a program with CUDA launches, stream
// events, peer stores and NCCL; kgs_step_program (kgs_host.cu) exports the
// same list so the multi-rank schedule can be replayed on the CPU against
// the oracle with real send/recv (tests/test_distributed_cpu.py).  No CUDA
// in here.
// Part of the single translation unit kgs_host.cu (included in order).
#pragma once

namespace {

enum ProgKind : int {
  PG_LAUNCH = 1,      // colour pass over local planes [xa, xb) of every slab
  PG_WAIT_XCH = 2,    // the slab's stream waits until the pending exchange landed
  PG_XCH = 3,         // start the exchange of colour `col` faces (P, Q, U of
                      // planes 0 and nx-1 -> the neighbours' ghost planes)
  PG_RECORD = 4,      // reduce the DIAG partials of the last passes into record `step`
                      // (xa = 1: both colours' partials)
  PG_DEFER = 5,       // the red adjoint of the last step is left pending
  PG_PASS_BEGIN = 6,  // a colour pass starts (xa = 1: timed as a fused pass)
  PG_PASS_END = 7,    // ... and ends
};

struct ProgOp {
  int kind = 0;
  int col = 0, op1 = OP_NONE, op2 = OP_NONE;  // colour; operations applied in order
  int diag = 0, check = 0;                    // energy terms; finiteness
  int step = 0;                               // step number (finiteness) / record slot
  int xa = 0, xb = 0;                         // plane range / flags (see ProgKind)
};
constexpr int kProgFields = 9;   // exported row: kind, col, op1, op2, diag, check, step, xa, xb

using Program = std::vector<ProgOp>;

// One colour pass.  A single slab (one GPU, one rank) wraps x inside the
// kernel: one launch.  Several slabs / ranks: the interior planes [1, nx-1)
// need no ghost data, so they run first and overlap the previous pass's
// exchange; then the stream waits for that exchange and the two boundary
// planes run.
void emit_pass(Program& p, int64_t nx, bool split, int col, int op1, int op2, bool diag,
               bool check, int step, bool timed) {
  ProgOp b;
  b.kind = PG_PASS_BEGIN;
  b.col = col; b.op1 = op1; b.op2 = op2; b.diag = diag; b.check = check; b.step = step;
  b.xa = timed ? 1 : 0;
  p.push_back(b);
  ProgOp l = b;
  l.kind = PG_LAUNCH;
  if (!split) {
    l.xa = 0; l.xb = (int)nx;
    p.push_back(l);
  } else {
    if (nx > 2) { l.xa = 1; l.xb = (int)nx - 1; p.push_back(l); }
    ProgOp w;
    w.kind = PG_WAIT_XCH;
    p.push_back(w);
    l.xa = 0; l.xb = 1;
    p.push_back(l);
    l.xa = (int)nx - 1; l.xb = (int)nx;
    p.push_back(l);
  }
  ProgOp e = b;
  e.kind = PG_PASS_END;
  p.push_back(e);
}

void emit_xch(Program& p, int col) {
  ProgOp x;
  x.kind = PG_XCH;
  x.col = col;
  p.push_back(x);
}

// Flags of a stepping call.  PGF_HEAD_FUSED: the previous call left its red
// adjoint pending with the SAME coefficients, so it fuses into this call's
// head (a pending adjoint with other coefficients is flushed before the
// program runs, as its own pass).  PGF_DEFER: leave this call's red
// adjoint tail pending (KGS_STEP_DEFER_TAIL) unless the last step records.
enum : int { PGF_HEAD_FUSED = 2, PGF_DEFER = 4 };

// kgs_step_dpavf2 (integrate's loop body, integrator.py:167-179, with the
// K3/K4 fusion of DESIGN.md §4):
//   head:  red base(first step) -- fused with a pending red adjoint of the
//          previous call when the coefficients match (PGF_HEAD_FUSED);
//   n:     K3 black base(n)+adjoint(n) | K4 red adjoint(n)+base(n+1)
//          (last step: the red adjoint tail, or left pending with PGF_DEFER);
//   every colour pass is followed by the exchange of the colour it wrote;
//   a record step reduces both passes' partials; the call ends when the last
//   exchange has landed.
Program step_program(int64_t nx, bool split, int64_t nsteps, int64_t step_offset,
                     int64_t record_stride, int flags) {
  Program p;
  if (nsteps <= 0) return p;
  const int64_t last = step_offset + nsteps;
  const bool defer = (flags & PGF_DEFER) && !(record_stride > 0 && last % record_stride == 0);
  if (flags & PGF_HEAD_FUSED)
    emit_pass(p, nx, split, 1, OP_ADJ, OP_BASE, false, false, 0, false);
  else
    emit_pass(p, nx, split, 1, OP_BASE, OP_NONE, false, false, 0, false);
  emit_xch(p, 1);
  int slot = 0;
  for (int64_t i = 1; i <= nsteps; ++i) {
    const int n = (int)(step_offset + i);
    const bool rec = record_stride > 0 && n % record_stride == 0;
    emit_pass(p, nx, split, 0, OP_BASE, OP_ADJ, rec, true, n, true);
    emit_xch(p, 0);
    if (i < nsteps) {
      emit_pass(p, nx, split, 1, OP_ADJ, OP_BASE, rec, true, n, true);
    } else if (defer) {
      ProgOp d;
      d.kind = PG_DEFER;
      p.push_back(d);
      break;
    } else {
      emit_pass(p, nx, split, 1, OP_ADJ, OP_NONE, rec, true, n, false);
    }
    emit_xch(p, 1);
    if (rec) {
      ProgOp r;
      r.kind = PG_RECORD;
      r.step = slot++;
      r.xa = 1;
      p.push_back(r);
    }
  }
  ProgOp w;
  w.kind = PG_WAIT_XCH;
  p.push_back(w);
  return p;
}

// One colour pass of colour `col` applying op1 then op2, followed by the
// exchange of the faces it wrote (kgs_sweep: one phase of step_base /
// step_adjoint, integrator.py:107-121; the energy passes; a pending tail).
Program pass_program(int64_t nx, bool split, int col, int op1, int op2, bool diag, bool check,
                     int step, bool xch) {
  Program p;
  emit_pass(p, nx, split, col, op1, op2, diag, check, step, false);
  if (xch) emit_xch(p, col);
  return p;
}

}  // namespace
