/*
 * svgrad_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).
 *
 * A plain-C restatement of the reference's reverse-mode schedule, following
 * it step by step with materialised states and the reference's primitive
 * semantics.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
 * may load this; the product (paper_2009_02823_b200) never does.
 *
 *   apply_matrix      <- svgrad/statevector.py:89-144  (group gather, m @ v, scatter;
 *                        sub-index bit k <-> targets[k]; controls all 1)
 *   project_to_one    <- svgrad/statevector.py:147-167
 *   clone / inner     <- svgrad/statevector.py:56-71   (np.vdot conjugates the bra)
 *   apply_observable  <- svgrad/observable.py:79-100   (per term: copy, non-I factors, axpy)
 *   oracle_sweep      <- svgrad/gradients.py:128-173   (_reverse_sweep, literal order:
 *                        forward, clone, observable, energy, then per gate i descending:
 *                        rewind ket; per local parameter clone a probe, apply the
 *                        derivative action, accumulate scalar*<bra|probe>; adjoint on bra if i>0)
 *   derivative action <- svgrad/circuit.py:302-334     (Pauli: sigma per axis then the bound
 *                        rotation; Phase: projection; matrix kinds: dM; then control projection)
 *
 * Parallelised with OpenMP over amplitude groups (static schedule, so a given
 * thread count gives bit-identical results).
 */
#include <complex.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

enum { DK_PAULI_ROTATION = 0, DK_PHASE = 1, DK_MATRIX = 2 };

typedef struct {
  int32_t num_qubits;
  int32_t num_gates;
  int32_t num_params;
  int32_t num_derivs;
  int32_t num_terms;
  int32_t num_threads;       /* 0 = OpenMP default */
  /* gates */
  const int32_t* ntargets;   /* [G] */
  const int32_t* targets;    /* [G*2] */
  const int32_t* ctrl_off;   /* [G+1] offsets into controls */
  const int32_t* controls;
  const cplx* fwd;           /* [G*16] row-major 2^k x 2^k */
  const cplx* rewind;        /* [G*16] */
  const cplx* adjoint;       /* [G*16] */
  const int32_t* arity;      /* [G] */
  /* derivative occurrences, gate-major */
  const int32_t* dkind;      /* [A] */
  const int32_t* daxes;      /* [A*2] Pauli index 1=X 2=Y 3=Z per target (DK_PAULI_ROTATION) */
  const cplx* dmat;          /* [A*16] rotation matrix (Pauli) or dM (matrix kinds) */
  const cplx* dscalar;       /* [A] deferred scalar (alpha*i, i*e^{i theta}, 1) incl. test scale */
  const int32_t* dref;       /* [A] parameter slot */
  /* observable */
  const cplx* tcoeff;        /* [T] */
  const int32_t* tf_off;     /* [T+1] offsets into factor arrays */
  const int32_t* tf_qubit;
  const cplx* tf_mat;        /* [F*4] 2x2 factor matrices */
  /* input */
  const cplx* input;         /* [2^n] */
} oracle_problem;

typedef struct {
  int64_t gate_applies, derivative_applies, clones, inner_products, observable_applies;
} oracle_counters;

static const cplx PAULI[4][4] = {
    {1, 0, 0, 1}, {0, 1, 1, 0}, {0, -I, I, 0}, {1, 0, 0, -1}};

static int cmp_int(const void* a, const void* b) { return *(const int*)a - *(const int*)b; }

/* Enumerate exactly the groups the reference's _group_indices table holds:
 * target bits 0, control bits 1, every other bit free (group id with zero
 * bits inserted at the sorted fixed positions). */
static void apply_matrix(cplx* amps, int n, const cplx* m, int nt, const int32_t* targets,
                         int nc, const int32_t* controls) {
  int64_t cmask = 0;
  int fixed[64];
  int nf = 0;
  for (int k = 0; k < nt; ++k) fixed[nf++] = targets[k];
  for (int k = 0; k < nc; ++k) {
    fixed[nf++] = controls[k];
    cmask |= (int64_t)1 << controls[k];
  }
  qsort(fixed, nf, sizeof(int), cmp_int);
  int64_t off[4] = {0, 0, 0, 0};
  for (int k = 0; k < nt; ++k) {
    const int64_t half = (int64_t)1 << k;
    for (int64_t s = 0; s < half; ++s) off[half + s] = off[s] + ((int64_t)1 << targets[k]);
  }
  const int g = 1 << nt;
  const int64_t groups = (int64_t)1 << (n - nf);
#pragma omp parallel for schedule(static)
  for (int64_t gi = 0; gi < groups; ++gi) {
    int64_t idx = gi;
    for (int f = 0; f < nf; ++f) {
      const int64_t low = idx & (((int64_t)1 << fixed[f]) - 1);
      idx = ((idx >> fixed[f]) << (fixed[f] + 1)) | low;
    }
    idx |= cmask;
    if (g == 2) {
      const cplx v0 = amps[idx], v1 = amps[idx + off[1]];
      amps[idx] = m[0] * v0 + m[1] * v1;
      amps[idx + off[1]] = m[2] * v0 + m[3] * v1;
      continue;
    }
    cplx v[4], w[4];
    for (int s = 0; s < g; ++s) v[s] = amps[idx + off[s]];
    for (int r = 0; r < g; ++r) {
      cplx acc = 0;
      for (int s = 0; s < g; ++s) acc += m[r * g + s] * v[s];
      w[r] = acc;
    }
    for (int r = 0; r < g; ++r) amps[idx + off[r]] = w[r];
  }
}

static void project_to_one(cplx* amps, int n, int nq, const int32_t* qubits) {
  const int64_t dim = (int64_t)1 << n;
  int64_t mask = 0;
  for (int k = 0; k < nq; ++k) mask |= (int64_t)1 << qubits[k];
  if (!mask) return;
#pragma omp parallel for schedule(static)
  for (int64_t idx = 0; idx < dim; ++idx)
    if ((idx & mask) != mask) amps[idx] = 0;
}

static void copy_state(cplx* dst, const cplx* src, int n) {
  const int64_t dim = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < dim; ++i) dst[i] = src[i];
}

static cplx inner(const cplx* bra, const cplx* ket, int n) {
  const int64_t dim = (int64_t)1 << n;
  double re = 0, im = 0;
#pragma omp parallel for schedule(static) reduction(+ : re, im)
  for (int64_t i = 0; i < dim; ++i) {
    const cplx z = conj(bra[i]) * ket[i];
    re += creal(z);
    im += cimag(z);
  }
  return re + I * im;
}

/* out = sum_t c_t (tensor factors) state;  svgrad/observable.py:79-100 */
static void apply_observable(const oracle_problem* p, const cplx* state, cplx* out, cplx* scratch) {
  const int n = p->num_qubits;
  const int64_t dim = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < dim; ++i) out[i] = 0;
  for (int t = 0; t < p->num_terms; ++t) {
    copy_state(scratch, state, n);
    for (int f = p->tf_off[t]; f < p->tf_off[t + 1]; ++f)
      apply_matrix(scratch, n, p->tf_mat + 4 * f, 1, p->tf_qubit + f, 0, NULL);
    const cplx c = p->tcoeff[t];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < dim; ++i) out[i] += c * scratch[i];
  }
}

int oracle_sweep(const oracle_problem* p, cplx* sums, cplx* energy, oracle_counters* cnt) {
#ifdef _OPENMP
  if (p->num_threads > 0) omp_set_num_threads(p->num_threads);
#endif
  const int n = p->num_qubits;
  const size_t bytes = sizeof(cplx) * ((size_t)1 << n);
  cplx* bra = malloc(bytes);
  cplx* ket = malloc(bytes);
  cplx* probe = malloc(bytes);
  cplx* obs = malloc(bytes);
  if (!bra || !ket || !probe || !obs) {
    free(bra); free(ket); free(probe); free(obs);
    return 1;
  }
  memset(cnt, 0, sizeof(*cnt));
  for (int q = 0; q < p->num_params; ++q) sums[q] = 0;

  copy_state(bra, p->input, n);  /* bra = clone_state(input) */
  cnt->clones++;
  for (int i = 0; i < p->num_gates; ++i) {
    apply_matrix(bra, n, p->fwd + 16 * i, p->ntargets[i], p->targets + 2 * i,
                 p->ctrl_off[i + 1] - p->ctrl_off[i], p->controls + p->ctrl_off[i]);
    cnt->gate_applies++;
  }
  copy_state(ket, bra, n);       /* ket = clone_state(bra) */
  cnt->clones++;
  apply_observable(p, bra, obs, probe);  /* bra = apply_observable(bra, obs) */
  cnt->observable_applies++;
  { cplx* t = bra; bra = obs; obs = t; }
  *energy = inner(ket, bra, n);  /* uncounted, as in the reference */

  int d_end = p->num_derivs;
  for (int i = p->num_gates - 1; i >= 0; --i) {
    const int nt = p->ntargets[i];
    const int32_t* tg = p->targets + 2 * i;
    const int nc = p->ctrl_off[i + 1] - p->ctrl_off[i];
    const int32_t* cg = p->controls + p->ctrl_off[i];
    const int d0 = d_end - p->arity[i];
    apply_matrix(ket, n, p->rewind + 16 * i, nt, tg, nc, cg);
    cnt->gate_applies++;
    for (int d = d0; d < d_end; ++d) {
      copy_state(probe, ket, n);
      cnt->clones++;
      if (p->dkind[d] == DK_PAULI_ROTATION) {
        for (int k = 0; k < nt; ++k) apply_matrix(probe, n, PAULI[p->daxes[2 * d + k]], 1, tg + k, 0, NULL);
        apply_matrix(probe, n, p->dmat + 16 * d, nt, tg, 0, NULL);
      } else if (p->dkind[d] == DK_PHASE) {
        project_to_one(probe, n, nt, tg);
      } else {
        apply_matrix(probe, n, p->dmat + 16 * d, nt, tg, 0, NULL);
      }
      if (nc) project_to_one(probe, n, nc, cg);
      cnt->derivative_applies++;
      sums[p->dref[d]] += p->dscalar[d] * inner(bra, probe, n);
      cnt->inner_products++;
    }
    d_end = d0;
    if (i > 0) {
      apply_matrix(bra, n, p->adjoint + 16 * i, nt, tg, nc, cg);
      cnt->gate_applies++;
    }
  }
  free(bra); free(ket); free(probe); free(obs);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Large-n variant of oracle_sweep (n = 30 fixtures on a host with tens of GiB):
 * the same schedule, counters and per-amplitude arithmetic, with two storage
 * economies that do not change any value the reference computes:
 *   - input given as a basis index (init_basis_state, svgrad/statevector.py:43-53)
 *     instead of a 2^n host array;
 *   - the derivative probe (clone + derivative action + projection + inner
 *     product, svgrad/gradients.py:161-165 with svgrad/circuit.py:302-334) is
 *     evaluated group by group instead of being materialised: for each group of
 *     the gate's targets the probe amplitudes are formed exactly as the
 *     materialised sequence forms them (sigma per axis as a 2x2 product, then the
 *     bound matrix, then the control projection) and contracted with the bra at
 *     once.  Only the order of the inner product's floating-point sum differs.
 *   - the observable is applied to ket (a clone of bra holding the same values),
 *     so the pre-observable bra is released first: peak 3 states, 2 in the sweep.
 * Checked against oracle_sweep on every golden case (tests/test_oracle.py).
 * ------------------------------------------------------------------------- */
static cplx deriv_inner(const oracle_problem* p, int d, const cplx* bra, const cplx* ket, int n, int nt,
                        const int32_t* tg, int nc, const int32_t* cg) {
  int64_t cmask = 0;
  for (int k = 0; k < nc; ++k) cmask |= (int64_t)1 << cg[k];
  int fixed[64];
  int nf = 0;
  for (int k = 0; k < nt; ++k) fixed[nf++] = tg[k];
  qsort(fixed, nf, sizeof(int), cmp_int);
  int64_t off[4] = {0, 0, 0, 0};
  for (int k = 0; k < nt; ++k) {
    const int64_t half = (int64_t)1 << k;
    for (int64_t s = 0; s < half; ++s) off[half + s] = off[s] + ((int64_t)1 << tg[k]);
  }
  const int g = 1 << nt;
  const int64_t groups = (int64_t)1 << (n - nf);
  const int kind = p->dkind[d];
  const cplx* dm = p->dmat + 16 * d;
  double re = 0, im = 0;
#pragma omp parallel for schedule(static) reduction(+ : re, im)
  for (int64_t gi = 0; gi < groups; ++gi) {
    int64_t idx = gi;
    for (int f = 0; f < nf; ++f) {
      const int64_t low = idx & (((int64_t)1 << fixed[f]) - 1);
      idx = ((idx >> fixed[f]) << (fixed[f] + 1)) | low;
    }
    cplx v[4], w[4];
    for (int s = 0; s < g; ++s) v[s] = ket[idx + off[s]];
    if (kind == DK_PAULI_ROTATION) {
      for (int k = 0; k < nt; ++k) {  /* sigma on target k: 1-target apply_matrix */
        const cplx* m = PAULI[p->daxes[2 * d + k]];
        const int b = 1 << k;
        for (int s = 0; s < g; ++s) {
          if (s & b) continue;
          const cplx v0 = v[s], v1 = v[s | b];
          v[s] = m[0] * v0 + m[1] * v1;
          v[s | b] = m[2] * v0 + m[3] * v1;
        }
      }
    }
    if (kind == DK_PHASE) {  /* project_to_one on the targets */
      for (int s = 0; s < g; ++s) w[s] = (s == g - 1) ? v[s] : 0;
    } else if (g == 2) {  /* the bound rotation / dM, as apply_matrix does it */
      w[0] = dm[0] * v[0] + dm[1] * v[1];
      w[1] = dm[2] * v[0] + dm[3] * v[1];
    } else {
      for (int r = 0; r < g; ++r) {
        cplx acc = 0;
        for (int s = 0; s < g; ++s) acc += dm[r * g + s] * v[s];
        w[r] = acc;
      }
    }
    if ((idx & cmask) != cmask) continue;  /* control projection: the probe is 0 here */
    for (int s = 0; s < g; ++s) {
      const cplx z = conj(bra[idx + off[s]]) * w[s];
      re += creal(z);
      im += cimag(z);
    }
  }
  return re + I * im;
}

int oracle_sweep_lean(const oracle_problem* p, int64_t basis, cplx* sums, cplx* energy, oracle_counters* cnt) {
#ifdef _OPENMP
  if (p->num_threads > 0) omp_set_num_threads(p->num_threads);
#endif
  const int n = p->num_qubits;
  const int64_t dim = (int64_t)1 << n;
  const size_t bytes = sizeof(cplx) * (size_t)dim;
  cplx* ket = malloc(bytes);
  if (!ket) return 1;
  memset(cnt, 0, sizeof(*cnt));
  for (int q = 0; q < p->num_params; ++q) sums[q] = 0;
  if (p->input) {
    copy_state(ket, p->input, n);
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < dim; ++i) ket[i] = 0;
    ket[basis] = 1;
  }
  cnt->clones++;  /* bra = clone_state(input) */
  for (int i = 0; i < p->num_gates; ++i) {
    apply_matrix(ket, n, p->fwd + 16 * i, p->ntargets[i], p->targets + 2 * i,
                 p->ctrl_off[i + 1] - p->ctrl_off[i], p->controls + p->ctrl_off[i]);
    cnt->gate_applies++;
  }
  cnt->clones++;  /* ket = clone_state(bra): same values, kept in `ket` */
  cplx* bra = malloc(bytes);
  cplx* scratch = malloc(bytes);
  if (!bra || !scratch) {
    free(ket); free(bra); free(scratch);
    return 1;
  }
  apply_observable(p, ket, bra, scratch);  /* bra = apply_observable(bra, obs) */
  cnt->observable_applies++;
  free(scratch);
  *energy = inner(ket, bra, n);

  int d_end = p->num_derivs;
  for (int i = p->num_gates - 1; i >= 0; --i) {
    const int nt = p->ntargets[i];
    const int32_t* tg = p->targets + 2 * i;
    const int nc = p->ctrl_off[i + 1] - p->ctrl_off[i];
    const int32_t* cg = p->controls + p->ctrl_off[i];
    const int d0 = d_end - p->arity[i];
    apply_matrix(ket, n, p->rewind + 16 * i, nt, tg, nc, cg);
    cnt->gate_applies++;
    for (int d = d0; d < d_end; ++d) {
      cnt->clones++;
      cnt->derivative_applies++;
      sums[p->dref[d]] += p->dscalar[d] * deriv_inner(p, d, bra, ket, n, nt, tg, nc, cg);
      cnt->inner_products++;
    }
    d_end = d0;
    if (i > 0) {
      apply_matrix(bra, n, p->adjoint + 16 * i, nt, tg, nc, cg);
      cnt->gate_applies++;
    }
  }
  free(bra); free(ket);
  return 0;
}

/* Per-primitive wall times (seconds) on 2^n states, for the op-count model of
 * oracle_sweep's cost (bench.py's CPU baseline): out[0] 1-target apply_matrix,
 * [1] 1-target with one control, [2] 2-target apply_matrix, [3] clone,
 * [4] inner product, [5] project_to_one (1 qubit), [6] observable axpy,
 * [7] observable zero fill. */
int oracle_time_primitives(int n, int threads, double* out) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  const int64_t dim = (int64_t)1 << n;
  const size_t bytes = sizeof(cplx) * (size_t)dim;
  cplx* a = malloc(bytes);
  cplx* b = malloc(bytes);
  if (!a || !b) {
    free(a); free(b);
    return 1;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < dim; ++i) {
    a[i] = (double)(i & 1023) * 1e-3 + I * 1e-3;
    b[i] = 0;
  }
  const double c = 0.8, s = 0.6;
  const cplx m1[4] = {c, -s, s, c};
  const cplx m2[16] = {c - I * s, 0, 0, 0, 0, c + I * s, 0, 0, 0, 0, c + I * s, 0, 0, 0, 0, c - I * s};
  const int32_t t1[1] = {n / 2}, t2[2] = {n / 2, n / 2 + 1}, ctl[1] = {n / 2 - 1};
  volatile double sink = 0;
  for (int k = 0; k < 8; ++k) {
    const double t0 = omp_get_wtime();
    switch (k) {
      case 0: apply_matrix(a, n, m1, 1, t1, 0, NULL); break;
      case 1: apply_matrix(a, n, m1, 1, t1, 1, ctl); break;
      case 2: apply_matrix(a, n, m2, 2, t2, 0, NULL); break;
      case 3: copy_state(b, a, n); break;
      case 4: sink += creal(inner(a, b, n)); break;
      case 5: project_to_one(b, n, 1, t1); break;
      case 6: {
        const cplx cc = 0.5;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < dim; ++i) b[i] += cc * a[i];
        break;
      }
      case 7: {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < dim; ++i) b[i] = 0;
        break;
      }
    }
    out[k] = omp_get_wtime() - t0;
  }
  (void)sink;
  free(a); free(b);
  return 0;
}

/* <psi|H|psi> after the forward pass only (svgrad/observable.py:114-116). */
int oracle_expectation(const oracle_problem* p, cplx* energy) {
#ifdef _OPENMP
  if (p->num_threads > 0) omp_set_num_threads(p->num_threads);
#endif
  const int n = p->num_qubits;
  const size_t bytes = sizeof(cplx) * ((size_t)1 << n);
  cplx* psi = malloc(bytes);
  cplx* out = malloc(bytes);
  cplx* scratch = malloc(bytes);
  if (!psi || !out || !scratch) {
    free(psi); free(out); free(scratch);
    return 1;
  }
  copy_state(psi, p->input, n);
  for (int i = 0; i < p->num_gates; ++i)
    apply_matrix(psi, n, p->fwd + 16 * i, p->ntargets[i], p->targets + 2 * i,
                 p->ctrl_off[i + 1] - p->ctrl_off[i], p->controls + p->ctrl_off[i]);
  apply_observable(p, psi, out, scratch);
  *energy = inner(psi, out, n);
  free(psi); free(out); free(scratch);
  return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
