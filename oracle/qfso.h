/* qfso.h — CPU ORACLE for QFactor-Sample instantiation (arXiv 2405.12866).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2405_12866_b200/csrc, include/qfs.h) and neither includes the other.
 *
 * Plain C++17, dense loops, double (re, im) arithmetic, long double
 * accumulation of environments and costs, no BLAS, no SIMD intrinsics, its own
 * one-sided Jacobi SVD.  Every function cites the PAPER.md passage it follows
 * (P:<line>); DESIGN.md §2 lists the readings taken where the paper is silent.
 *
 * Conventions (readings 1-4): complex numbers are double[2]
 * interleaved (re, im); amplitude index little-endian (bit q = qubit q); a gate
 * on the ordered pair (p0, p1) acts on l = b(p0) + 2 b(p1); matrices row-major
 * [row][col]; gates G[l_out][l_in]; states row-major [m][2^n].
 *
 * Return values: 0 on success, nonzero on argument error (no exceptions).
 */
#ifndef QFSO_H
#define QFSO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double dist_tol;        /* success threshold on c_train            */
  double diff_tol_r;      /* plateau relative improvement        */
  int plateau_window;     /* plateau window; <= 0 disables           */
  int min_iter;
  int max_iter;           /* total sweeps incl. restarts             */
  int m_init;             /* number_of_training_states               */
  double overtrain_ratio; /* P:368-372; +inf disables the gen. check         */
  double beta;
  int stop_on_first;      /* stop every start at the first converged sweep   */
} qfso_params;

typedef struct {
  double c_train, c_val;
  int sweeps, restarts, final_m, term; /* term: 0 CONVERGED 1 PLATEAU 2 MAX_ITER
                                          3 POOL_EXHAUSTED 4 STOPPED */
} qfso_result;

/* apply one 4x4 gate (or its adjoint when dagger != 0) to m states in place. P:59 */
int qfso_apply_gate(int n, int p0, int p1, const double *g, int dagger, int m, double *psi);
/* psi <- G_{K-1} ... G_0 psi (gate 0 first; reading 2). P:127 (B tensors) */
int qfso_circuit_forward(int n, int k, const int32_t *pairs, const double *gates, int m,
                         double *psi);
/* E[l_in][l_out] = sum_m sum_r phi_m[idx_r(l_in)] conj(chi_m[idx_r(l_out)]). P:121-125 */
int qfso_environment(int n, int p0, int p1, int m, const double *phi, const double *chi,
                     double *env);
/* one-sided (Hestenes) Jacobi SVD a = x diag(sigma) y^dag (sigma NOT sorted). P:59-62 */
int qfso_svd4(const double *a, double *x, double *sigma, double *y, int *sweeps);
/* g_new = Y X^dag from SVD((1-beta) E + beta g_old^dag); *sigma_sum = sum sigma. P:59-62 */
int qfso_polar_update(const double *env, const double *g_old, double beta, double *g_new,
                      double *sigma_sum);
/* scaled Newton polar iteration; w = unitary polar factor of a (a = w h). self-check only */
int qfso_newton_polar(const double *a, double *w, int *iters);
/* (1/m) sum_m ||a_m - b_m||^2 (direct distance form of P:116-120; reading 6) */
double qfso_distance(int n, int m, const double *a, const double *b);

/* Run n_sweeps sweeps at fixed M (first M pool rows) for s starts, no controller.
 * traces (any may be NULL):
 *   env_trace   [n_sweeps][k][s][4][4][2]  E_i as seen at gate i of sweep t
 *   gate_trace  [n_sweeps][s][k][4][4][2]  gates after sweep t
 *   cost_trace  [n_sweeps][s]              c_train after sweep t (direct form)
 *   sigma_trace [n_sweeps][k][s]           sum of singular values at gate i
 * shards: g >= 1.  g > 1 emulates sample sharding: rows m with m mod g == r form
 * shard r; partial environments / cost sums are formed per shard and summed in
 * rank order. */
int qfso_trace_sweeps(int n, int k, const int32_t *pairs, int s, const double *init_gates, int m,
                      const double *x, const double *y, double beta, int n_sweeps, int g,
                      double *env_trace, double *gate_trace, double *cost_trace,
                      double *sigma_trace, int n_threads);

/* Same with gate kinds (kinds[k]: 0 two-qubit variable block, 1 fixed gate,
 * 2 one-qubit variable gate u on the pair's first qubit, stored as u (x) I;
 * NULL = all 0).  SURVEY.md §8(f) NEXT-3; readings R24-R25. */
int qfso_trace_sweeps_kinds(int n, int k, const int32_t *pairs, const int32_t *kinds, int s,
                            const double *init_gates, int m, const double *x, const double *y,
                            double beta, int n_sweeps, int g, double *env_trace, double *gate_trace,
                            double *cost_trace, double *sigma_trace, int n_threads);

/* Full instantiation with the controller. */
int qfso_instantiate(int n, int k, const int32_t *pairs, int m_pool, const double *x,
                     const double *y, int v, const double *xv, const double *yv, int s,
                     const double *init_gates, const qfso_params *p, double *out_gates,
                     qfso_result *out, int *winner, int n_threads);

int qfso_instantiate_kinds(int n, int k, const int32_t *pairs, const int32_t *kinds, int m_pool,
                           const double *x, const double *y, int v, const double *xv,
                           const double *yv, int s, const double *init_gates, const qfso_params *p,
                           double *out_gates, qfso_result *out, int *winner, int n_threads);

/* Multi-qubit blocks ("possibly multi-qubit"
 * gates).  Gate k has arity a_k in {2, 3} on qubits[3k .. 3k+a_k-1] (as given;
 * local index l = sum_j b(q_j) 2^j), a d_k x d_k matrix G[l_out][l_in],
 * d_k = 2^a_k.  Gates are PACKED: gate k of start s at complex offset
 * s * G + off_k, off_k = sum_{j<k} d_j^2, G = off_K.  kinds as above (2 only
 * for arity 2; NULL = all variable).  env_trace per sweep t is gate-major:
 * gate i of start s at t * S * G + S * off_i + s * d_i^2. */
int qfso_apply_block(int n, int arity, const int32_t *q, const double *g, int dagger, int m, double *psi);
int qfso_environment_block(int n, int arity, const int32_t *q, int m, const double *phi,
                           const double *chi, double *env);
/* d in {4, 8}: g_new = Y X^dag from SVD((1-beta) E + beta g_old^dag), *sigma_sum = sum sigma */
int qfso_polar_update_block(int d, const double *env, const double *g_old, double beta, double *g_new,
                            double *sigma_sum);
int qfso_trace_sweeps_blocks(int n, int k, const int32_t *qubits, const int32_t *arity, const int32_t *kinds,
                             int s, const double *init_gates, int m, const double *x, const double *y,
                             double beta, int n_sweeps, double *env_trace, double *gate_trace,
                             double *cost_trace, double *sigma_trace, int n_threads);
int qfso_instantiate_blocks(int n, int k, const int32_t *qubits, const int32_t *arity, const int32_t *kinds,
                            int m_pool, const double *x, const double *y, int v, const double *xv,
                            const double *yv, int s, const double *init_gates, const qfso_params *p,
                            double *out_gates, qfso_result *out, int *winner, int n_threads);

/* Sweep-throughput timing: n_sweeps sweeps at fixed M; *sec = wall seconds. */
int qfso_bench_sweeps(int n, int k, const int32_t *pairs, int s, const double *init_gates, int m,
                      const double *x, const double *y, int n_sweeps, int n_threads,
                      double *sec);

#ifdef __cplusplus
}
#endif
#endif
