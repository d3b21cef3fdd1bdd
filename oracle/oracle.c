/*
 * oracle.c — plain, slow, fp64 CPU oracle for exact multi-head self-attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this file.  It shares no
 * code, header, table or helper with the CUDA path (paper_2405_15780_b200/), and
 * neither side includes or imports the other.
 *
 * What it computes (the plain definition the method reaches up to rounding):
 *   PAPER.md P:165 (§2.5, "Sequence Parallel (SP)"): after the all-to-all each GPU
 *     holds "a complete sequence, but only for a non-overlapping subset of the
 *     attention heads" and computes ordinary attention for those heads.
 *   PAPER.md P:173-175 (§2.6, "Flash Attention v2"): FlashAttention tiles the
 *     attention matrix; it is exact, so its result is the dense definition.
 *   SPEC.md S:176 (mha_forward): out_h = softmax(Q_h K_h^T * scale) V_h,
 *     scale = 1/sqrt(d_h); S:181-183 (mha_backward, analytic gradients);
 *     S:188 (the tiled forward also returns the per-row logsumexp);
 *     S:211-212 (no causal mask, no bias).
 *
 * Definitions, per batch b, head h, query row i, key row j (no blocking, no
 * online rescaling — a two-pass max/sum per row):
 *   s_ij  = scale * sum_d q[i,d] k[j,d]
 *   m_i   = max_j s_ij
 *   l_i   = sum_j exp(s_ij - m_i)
 *   lse_i = m_i + ln l_i                    (natural log of the scaled scores)
 *   P_ij  = exp(s_ij - lse_i)
 *   o_i   = sum_j P_ij v_j
 * Backward (standard softmax-attention calculus):
 *   dV_j  = sum_i P_ij dO_i
 *   dP_ij = dO_i . v_j
 *   Delta_i = dO_i . o_i                    (with the oracle's own fp64 o_i)
 *   dS_ij = P_ij (dP_ij - Delta_i)
 *   dQ_i  = scale sum_j dS_ij k_j
 *   dK_j  = scale sum_i dS_ij q_i
 *
 * Layouts (all contiguous, row-major, fp64):
 *   q, out, dout, dq          [B][Nq][H][D]
 *   k, v, dk, dv              [B][Nk][H][D]
 *   lse                       [B][H][Nq]
 * Self-attention is Nq == Nk; Nq != Nk serves the segment (LSS) tests, where a
 * query block attends to a contiguous key segment only.
 *
 * Parity pins live in tests/test_oracle.py (brute force, finite differences,
 * closed forms, invariants).  Every function here is pinned.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static double dot(const double* a, const double* b, int64_t D) {
  double acc = 0.0;
  for (int64_t d = 0; d < D; ++d) acc += a[d] * b[d];
  return acc;
}

/* Thread count of the OpenMP loops (harness plumbing, no arithmetic): the bench's
 * reference arm runs alone on rank 0 under torchrun, which sets OMP_NUM_THREADS=1. */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Forward for one query vector qi against keys/values of one (b, h).
 * kb/vb point at key 0 of that (b, h); consecutive keys are rs = H*D apart.
 * s is caller scratch of length Nk.  Writes o (D values) and returns lse.
 * If oabs != NULL it also writes sum_j P_ij |v_jd| — not part of the method:
 * the magnitude a rounding error in P_ij is multiplied by, used by the tests
 * to scale elementwise tolerances (equals o when V >= 0). */
static double attend_row(const double* qi, const double* kb, const double* vb,
                         int64_t Nk, int64_t rs, int64_t D, double scale,
                         double* s, double* o, double* oabs) {
  double m = -INFINITY;
  int64_t j = 0;
  /* Four keys at a time: four independent dot products, each summed over d in
   * the same order as dot() (bitwise-identical scores; only the instruction
   * schedule differs, so the loop is not bound by one add-latency chain). */
  for (; j + 4 <= Nk; j += 4) {
    const double* k0 = kb + j * rs;
    const double* k1 = k0 + rs;
    const double* k2 = k1 + rs;
    const double* k3 = k2 + rs;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int64_t d = 0; d < D; ++d) {
      a0 += qi[d] * k0[d];
      a1 += qi[d] * k1[d];
      a2 += qi[d] * k2[d];
      a3 += qi[d] * k3[d];
    }
    s[j] = scale * a0;
    s[j + 1] = scale * a1;
    s[j + 2] = scale * a2;
    s[j + 3] = scale * a3;
  }
  for (; j < Nk; ++j) s[j] = scale * dot(qi, kb + j * rs, D);
  for (j = 0; j < Nk; ++j)
    if (s[j] > m) m = s[j];
  double l = 0.0;
  for (j = 0; j < Nk; ++j) l += exp(s[j] - m);
  double lse = m + log(l);
  for (int64_t d = 0; d < D; ++d) o[d] = 0.0;
  if (oabs)
    for (int64_t d = 0; d < D; ++d) oabs[d] = 0.0;
  for (j = 0; j < Nk; ++j) {
    double p = exp(s[j] - lse);
    const double* vj = vb + j * rs;
    for (int64_t d = 0; d < D; ++d) o[d] += p * vj[d];
    if (oabs)
      for (int64_t d = 0; d < D; ++d) oabs[d] += p * fabs(vj[d]);
  }
  return lse;
}

/* Dense forward: out [B][Nq][H][D], lse [B][H][Nq]; out_abs (nullable)
 * [B][Nq][H][D] receives sum_j P_ij |v_jd| (see attend_row). */
void oracle_attn_fwd(const double* q, const double* k, const double* v,
                     int64_t B, int64_t Nq, int64_t Nk, int64_t H, int64_t D,
                     double* out, double* lse, double* out_abs) {
  const double scale = 1.0 / sqrt((double)D);
  const int64_t rs = H * D;
  const int64_t total = B * H * Nq;
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(Nk > 0 ? Nk : 1));
#pragma omp for schedule(static)
    for (int64_t t = 0; t < total; ++t) {
      int64_t b = t / (H * Nq), h = (t / Nq) % H, i = t % Nq;
      const double* qi = q + ((b * Nq + i) * H + h) * D;
      const double* kb = k + (b * Nk * H + h) * D;
      const double* vb = v + (b * Nk * H + h) * D;
      double* oi = out + ((b * Nq + i) * H + h) * D;
      double* ai = out_abs ? out_abs + ((b * Nq + i) * H + h) * D : NULL;
      lse[(b * H + h) * Nq + i] = attend_row(qi, kb, vb, Nk, rs, D, scale, s, oi, ai);
    }
    free(s);
  }
}

/* Forward for an explicit list of R query vectors.  qrows [R][D]; row r belongs
 * to (batch bh[2r], head bh[2r+1]) of k, v [B][Nk][H][D].  out_rows [R][D],
 * lse_rows [R].  Each o_i depends only on q_i, K and V, so this is the exact
 * forward for those rows (used for sampled checks at large N). */
void oracle_attn_fwd_rows(const double* qrows, const int64_t* bh, int64_t R,
                          const double* k, const double* v,
                          int64_t B, int64_t Nk, int64_t H, int64_t D,
                          double* out_rows, double* lse_rows) {
  (void)B;
  const double scale = 1.0 / sqrt((double)D);
  const int64_t rs = H * D;
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(Nk > 0 ? Nk : 1));
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
      int64_t b = bh[2 * r], h = bh[2 * r + 1];
      const double* kb = k + (b * Nk * H + h) * D;
      const double* vb = v + (b * Nk * H + h) * D;
      lse_rows[r] = attend_row(qrows + r * D, kb, vb, Nk, rs, D, scale, s, out_rows + r * D, NULL);
    }
    free(s);
  }
}

/* Dense backward (self-attention, Nq == Nk == N).  Recomputes the forward in
 * fp64 (pass 1), then dQ by rows (pass 2), then dK, dV by keys (pass 3) so no
 * two threads write the same output.  out/lse receive the fp64 forward.
 * gabs (nullable, [3][B][N][H][D]) receives the error-scale sums the tests use
 * for elementwise tolerances — not part of the method:
 *   gabs[0] = scale sum_j (|dS_ij| + P_ij e_i) |k_j|,
 *   gabs[1] = scale sum_i (|dS_ij| + P_ij e_i) |q_i|,
 *   gabs[2] = sum_i P_ij |dO_i|,     e_i = sum_d |dO_id o_id|
 * (the magnitudes that bf16 rounding of dS, P and of o inside Delta hits). */
void oracle_attn_bwd(const double* q, const double* k, const double* v,
                     const double* dout, int64_t B, int64_t N, int64_t H, int64_t D,
                     double* dq, double* dk, double* dv, double* out, double* lse,
                     double* gabs) {
  const double scale = 1.0 / sqrt((double)D);
  const int64_t rs = H * D;
  const int64_t total = B * H * N;
  const int64_t nel = B * N * H * D;
  double* delta = (double*)malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));
  /* edelta_i = sum_d |dO_id o_id|: the size of the perturbation of Delta_i when
   * o is rounded (error-scale helper only; used when gabs != NULL). */
  double* edelta = (double*)malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));

  /* pass 1: forward, and Delta_i = dO_i . o_i */
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
#pragma omp for schedule(static)
    for (int64_t t = 0; t < total; ++t) {
      int64_t b = t / (H * N), h = (t / N) % H, i = t % N;
      const int64_t ro = ((b * N + i) * H + h) * D;
      const double* kb = k + (b * N * H + h) * D;
      const double* vb = v + (b * N * H + h) * D;
      lse[(b * H + h) * N + i] = attend_row(q + ro, kb, vb, N, rs, D, scale, s, out + ro, NULL);
      delta[(b * H + h) * N + i] = dot(dout + ro, out + ro, D);
      double e = 0.0;
      for (int64_t d = 0; d < D; ++d) e += fabs(dout[ro + d] * out[ro + d]);
      edelta[(b * H + h) * N + i] = e;
    }
    free(s);
  }

  /* pass 2: dQ_i = scale * sum_j P_ij (dO_i . v_j - Delta_i) k_j */
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < total; ++t) {
    int64_t b = t / (H * N), h = (t / N) % H, i = t % N;
    const int64_t ro = ((b * N + i) * H + h) * D;
    const double li = lse[(b * H + h) * N + i];
    const double di = delta[(b * H + h) * N + i];
    double* dqi = dq + ro;
    double* aq = gabs ? gabs + ro : NULL;
    for (int64_t d = 0; d < D; ++d) dqi[d] = 0.0;
    if (aq)
      for (int64_t d = 0; d < D; ++d) aq[d] = 0.0;
    for (int64_t j = 0; j < N; ++j) {
      const double* kj = k + ((b * N + j) * H + h) * D;
      const double* vj = v + ((b * N + j) * H + h) * D;
      double p = exp(scale * dot(q + ro, kj, D) - li);
      double ds = p * (dot(dout + ro, vj, D) - di);
      for (int64_t d = 0; d < D; ++d) dqi[d] += ds * kj[d];
      if (aq)
        for (int64_t d = 0; d < D; ++d) aq[d] += (fabs(ds) + p * edelta[(b * H + h) * N + i]) * fabs(kj[d]);
    }
    for (int64_t d = 0; d < D; ++d) dqi[d] *= scale;
    if (aq)
      for (int64_t d = 0; d < D; ++d) aq[d] *= scale;
  }

  /* pass 3: dV_j = sum_i P_ij dO_i ; dK_j = scale * sum_i dS_ij q_i */
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < total; ++t) {
    int64_t b = t / (H * N), h = (t / N) % H, j = t % N;
    const int64_t rj = ((b * N + j) * H + h) * D;
    double* dkj = dk + rj;
    double* dvj = dv + rj;
    double* ak = gabs ? gabs + nel + rj : NULL;
    double* av = gabs ? gabs + 2 * nel + rj : NULL;
    for (int64_t d = 0; d < D; ++d) { dkj[d] = 0.0; dvj[d] = 0.0; }
    if (ak)
      for (int64_t d = 0; d < D; ++d) { ak[d] = 0.0; av[d] = 0.0; }
    for (int64_t i = 0; i < N; ++i) {
      const int64_t ri = ((b * N + i) * H + h) * D;
      double p = exp(scale * dot(q + ri, k + rj, D) - lse[(b * H + h) * N + i]);
      double ds = p * (dot(dout + ri, v + rj, D) - delta[(b * H + h) * N + i]);
      for (int64_t d = 0; d < D; ++d) {
        dvj[d] += p * dout[ri + d];
        dkj[d] += ds * q[ri + d];
      }
      if (ak)
        for (int64_t d = 0; d < D; ++d) {
          ak[d] += (fabs(ds) + p * edelta[(b * H + h) * N + i]) * fabs(q[ri + d]);
          av[d] += p * fabs(dout[ri + d]);
        }
    }
    for (int64_t d = 0; d < D; ++d) dkj[d] *= scale;
    if (ak)
      for (int64_t d = 0; d < D; ++d) ak[d] *= scale;
  }
  free(delta);
  free(edelta);
}

/* dQ for an explicit list of R query rows (exact, per row):
 *   P_ij = exp(s_ij - lse_i), Delta_i = dO_i . o_i with o_i, lse_i from the
 *   row's own forward, dQ_i = scale sum_j P_ij (dO_i . v_j - Delta_i) k_j.
 * qrows, dorows [R][D]; bh [R][2] = (batch, head) into k, v [B][Nk][H][D].
 * Writes dq_rows [R][D].  Used for sampled backward checks at large N. */
void oracle_attn_bwd_dq_rows(const double* qrows, const double* dorows, const int64_t* bh, int64_t R,
                             const double* k, const double* v, int64_t B, int64_t Nk, int64_t H, int64_t D,
                             double* dq_rows) {
  (void)B;
  const double scale = 1.0 / sqrt((double)D);
  const int64_t rs = H * D;
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(Nk > 0 ? Nk : 1));
    double* o = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
      const int64_t b = bh[2 * r], h = bh[2 * r + 1];
      const double* kb = k + (b * Nk * H + h) * D;
      const double* vb = v + (b * Nk * H + h) * D;
      const double* qi = qrows + r * D;
      const double* doi = dorows + r * D;
      const double lse = attend_row(qi, kb, vb, Nk, rs, D, scale, s, o, NULL);
      const double delta = dot(doi, o, D);
      double* dqi = dq_rows + r * D;
      for (int64_t d = 0; d < D; ++d) dqi[d] = 0.0;
      for (int64_t j = 0; j < Nk; ++j) {
        const double p = exp(s[j] - lse);
        const double ds = p * (dot(doi, vb + j * rs, D) - delta);
        for (int64_t d = 0; d < D; ++d) dqi[d] += ds * kb[j * rs + d];
      }
      for (int64_t d = 0; d < D; ++d) dqi[d] *= scale;
    }
    free(s);
    free(o);
  }
}

/* Exact dK_j, dV_j for R explicit key rows of ONE head (full-size parity of the
 * backward at sizes where the dense backward is out of reach).  qh, kh, vh, doh
 * are that head's [N][D] rows (self-attention, N queries = N keys).  Follows the
 * definitions above in order: pass 1 recomputes, for every query i, lse_i and
 * o_i (attend_row, the oracle's own fp64 forward) and Delta_i = dO_i . o_i;
 * then for each requested key j:
 *   dV_j = sum_i P_ij dO_i,  dK_j = scale sum_i P_ij (dO_i . v_j - Delta_i) q_i,
 * with P_ij = exp(s_ij - lse_i), s_ij = scale q_i . k_j. */
void oracle_attn_bwd_kv_rows(const double* qh, const double* kh, const double* vh, const double* doh, int64_t N,
                             int64_t D, const int64_t* keys, int64_t R, double* dk_rows, double* dv_rows) {
  const double scale = 1.0 / sqrt((double)D);
  double* lse = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  double* delta = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    double* o = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic, 16)
    for (int64_t i = 0; i < N; ++i) {
      lse[i] = attend_row(qh + i * D, kh, vh, N, D, D, scale, s, o, NULL);
      delta[i] = dot(doh + i * D, o, D);
    }
    free(s);
    free(o);
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < R; ++r) {
    const int64_t j = keys[r];
    const double* kj = kh + j * D;
    const double* vj = vh + j * D;
    double* dk = dk_rows + r * D;
    double* dv = dv_rows + r * D;
    for (int64_t d = 0; d < D; ++d) dk[d] = dv[d] = 0.0;
    for (int64_t i = 0; i < N; ++i) {
      const double* qi = qh + i * D;
      const double* doi = doh + i * D;
      const double p = exp(scale * dot(qi, kj, D) - lse[i]);
      const double ds = p * (dot(doi, vj, D) - delta[i]);
      for (int64_t d = 0; d < D; ++d) {
        dv[d] += p * doi[d];
        dk[d] += ds * qi[d];
      }
    }
    for (int64_t d = 0; d < D; ++d) dk[d] *= scale;
  }
  free(lse);
  free(delta);
}
