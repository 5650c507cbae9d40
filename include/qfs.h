/* qfs.h — C ABI of the B200-native QFactor-Sample instantiation library
 * (libqfs.so, arXiv 2405.12866).
 *
 * The library fits the 4x4 unitaries of a circuit of two-qubit blocks to a
 * target U from sampled input/output states (§3): each
 * sweep runs right to left over the gates, forms each gate's 4x4
 * environment E over all 2^n amplitudes and M samples,
 * replaces the gate by the unitary polar factor u = Y X^dag of E = X D Y^dag
 * (eq:opt_u), and a host controller grows M ("double-and-restart",
 * P:114) when the validation cost exceeds the training cost by
 * more than overtrain_ratio.  Every step of a sweep runs in
 * hand-written sm_100a CUDA kernels; there is no CPU fallback.
 *
 * Conventions (DESIGN.md §2 readings R1-R4):
 *  - complex numbers are double[2] interleaved (re, im) (std::complex<double>,
 *    cuDoubleComplex, numpy complex128 layout);
 *  - amplitude index is little-endian: bit q of the index is qubit q;
 *  - a gate on the ordered pair (p0, p1) acts on the local index
 *    l = b(p0) + 2*b(p1); gate matrices are row-major G[l_out][l_in];
 *  - gate 0 is applied first (nearest the input); C = G_{K-1} ... G_0;
 *  - states are row-major [row][2^n]; gates [start][gate][4][4].
 *
 * Ownership: the caller owns every host buffer; qfs_set_samples COPIES its
 * inputs (the caller may free them on return); the context owns all device
 * memory until qfs_destroy.  A context is not thread-safe; distinct contexts
 * are independent.  Errors are status codes only (no exceptions or exit cross
 * the ABI); qfs_last_error(ctx) returns the message of the last failure.
 */
#ifndef QFS_H
#define QFS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct qfs_ctx qfs_ctx; /* opaque; owns all device memory */

typedef enum {
  QFS_OK = 0,
  QFS_ERR_ARG = 1,      /* n < 2, p0 == p1, p >= n, k < 1, null pointer, bad count */
  QFS_ERR_CAPACITY = 2, /* m_init > m_pool, m_pool > 2^n, memory plan exceeds the device,
                           M not divisible by world in sample mode */
  QFS_ERR_NUMERIC = 3,  /* non-finite input, or initial gate not unitary (||G^dag G - I||_max > 1e-10) */
  QFS_ERR_DEVICE = 4,   /* CUDA / NCCL failure (message in qfs_last_error) */
  QFS_ERR_STATE = 5     /* instantiate / trace before set_samples */
} qfs_status;

typedef enum {
  QFS_CONVERGED = 0,      /* c_train <= dist_tol and generalisation check passed  */
  QFS_PLATEAU = 1,        /* plateau_window consecutive non-improving sweeps */
  QFS_MAX_ITER = 2,       /* total sweeps reached max_iter                      */
  QFS_POOL_EXHAUSTED = 3, /* overtrain needed 2M rows but the pool is smaller (M < 2^n)  */
  QFS_STOPPED = 4         /* stop_on_first: another start converged first                */
} qfs_term;

/* Hyperparameters of PAPER.md App. A. */
typedef struct {
  double dist_tol;        /* converged when c_train <= dist_tol (R8)             */
  double diff_tol_r;      /* plateau: |c_prev| - |c| > diff_tol_r |c| is progress */
  int plateau_window;     /* consecutive failures before PLATEAU; <= 0 disables */
  int min_iter;           /* no PLATEAU / overtrain stop before it (R9)          */
  int max_iter;           /* total sweeps across restarts                       */
  int m_init;             /* number_of_training_states                          */
  double overtrain_ratio; /* restart with 2M when c_val/c_train - 1 > otr;
                             +INFINITY disables the generalisation check                */
  double beta;            /* SVD of (1-beta) E + beta u^dag                 */
  int stop_on_first;      /* 1: stop all starts at the first sweep where one converged  */
} qfs_params;

typedef struct {
  double c_train, c_val; /* last training cost (direct form; R6) and validation cost */
  int sweeps, restarts, final_m;
  qfs_term term;
} qfs_result;

/* Create a context for an n-qubit circuit of k two-qubit blocks.
 * pairs: host int32 [k][2] (ordered qubit pairs; p0 != p1, both < n).
 * device: CUDA ordinal.  Structure only; no target. */
qfs_status qfs_create(int n, int k, const int32_t *pairs, int device, qfs_ctx **out);

/* Create a context for an n-qubit circuit of k multi-qubit blocks (SURVEY.md
 * §8(f) NEXT-3; "possibly multi-qubit" unitary gates).
 * qubits: host int32 [k][3]; block i acts on qubits[3i .. 3i+arity[i]-1] (distinct,
 * < n; entry 3i+2 ignored for arity 2), local index l = sum_j b(q_j) 2^j.
 * arity: host int32 [k], each 2 or 3.  Gate i is a d x d matrix G[l_out][l_in],
 * d = 2^arity[i].  GATE LAYOUT of every call of this context (init_gates,
 * out_gates, gate_trace): PACKED per start — gate i at complex offset
 * off_i = sum_{j<i} d_j^2 of the start's block of G = off_k entries
 * (all-two-qubit circuits: G = 16 k, the same layout as qfs_create, and the
 * context IS a pair context).  env_trace per sweep: gate-major, gate i of start
 * s at s_total * off_i + s * d_i^2.  Circuits with a 3-qubit block run the
 * streamed sweep (B cache in HBM) with one launch per step, single GPU
 * (qfs_create_dist / sample sharding are not available for them); the 8x8
 * update is the Newton-Schulz polar factor, with a one-sided Jacobi SVD for
 * singular or very ill-conditioned environments (null columns completed as
 * in the oracle; the gate is then not unique, only the cost is).  Gate
 * kinds (qfs_set_gate_kinds) apply per block: VAR2 = variable (any arity),
 * FIXED, VAR1 only on two-qubit blocks.  Errors: QFS_ERR_ARG for a bad
 * structure (n < 3, arity not 2/3, repeated or out-of-range qubits). */
qfs_status qfs_create_blocks(int n, int k, const int32_t *qubits, const int32_t *arity, int device,
                             qfs_ctx **out);

/* Replace the circuit structure of a pair context (same n): k gates on pairs
 * [k][2].  Samples, device buffers and streams are kept (re-planned only when
 * k exceeds what they were sized for); gate kinds reset to all QFS_GATE_VAR2;
 * the cached sweep graph is dropped.  For re-instantiating many structures on
 * the same samples (the gate-deletion flow) without a context per
 * structure.  Waits for the context's in-flight work.  Errors: QFS_ERR_ARG
 * (bad pairs, block context). */
qfs_status qfs_set_structure(qfs_ctx *c, int k, const int32_t *pairs);

/* Distributed context.  nccl_comm: an ncclComm_t whose rank
 * and size equal (rank, world) (e.g. ProcessGroupNCCL._comm_ptr()), or NULL
 * when world == 1.  shard_mode 0 = multistart (each rank runs its own starts,
 * no data-path collective); 1 = sample (each rank holds rows m = rank mod world
 * of the pool, passed LOCALLY to set_samples; partial environments and cost
 * sums are all-reduced per gate / per sweep over NCCL). */
qfs_status qfs_create_dist(int n, int k, const int32_t *pairs, int device, void *nccl_comm,
                           int rank, int world, int shard_mode, qfs_ctx **out);

/* Exchange of the partial environments in sample mode (
 * E is a sum over samples, so the ranks' partials add up):
 *   0 = host-enqueued ncclAllReduce of E per gate, then a separate polar launch
 *       (default);
 *   1 = device-initiated: the last CTA of each start's environment reduction
 *       stores its partial E into every rank's mailbox (CUDA-IPC-mapped peer
 *       memory over NVLink), raises an epoch flag there, waits for all ranks'
 *       flags and sums the partials in rank order, then runs the polar update
 *       itself — one launch per gate, no host involvement, identical bits on
 *       all ranks.
 * Collective in sample mode with world > 1 (the mailboxes are set up with the
 * context's NCCL communicator at the next call); QFS_ERR_STATE without one,
 * QFS_ERR_ARG for another value, a block context, or more than 32 ranks. */
qfs_status qfs_set_exchange(qfs_ctx *c, int mode);

/* Sample mode with `ranks` (2..32) EMULATED ranks on one device, for testing
 * and measuring the device-initiated exchange where fewer GPUs than ranks
 * exist: rank r holds pool rows m = r (mod ranks) (the caller passes ALL rows
 * to set_samples; m_pool divisible by ranks) with its own states and gate
 * copy; all ranks run in the same launches and exchange E through local
 * mailboxes with exactly the protocol of qfs_set_exchange(c, 1).  Every rank
 * evaluates the full validation set.  One start per call (s == 1, else
 * QFS_ERR_ARG).  Results equal the single-rank sweep up to the summation
 * order of E. */
qfs_status qfs_create_emulated(int n, int k, const int32_t *pairs, int device, int ranks, qfs_ctx **out);

/* NCCL bootstrap owned by the library: rank 0 calls qfs_nccl_unique_id
 * (128 opaque bytes), the caller broadcasts them (e.g. torch.distributed), and
 * every rank calls qfs_create_nccl; the context creates and owns the
 * communicator (destroyed by qfs_destroy).  Same semantics as qfs_create_dist. */
qfs_status qfs_nccl_unique_id(void *id128);
qfs_status qfs_create_nccl(int n, int k, const int32_t *pairs, int device, const void *id128,
                           int rank, int world, int shard_mode, qfs_ctx **out);

/* Training pool x, targets y = U x (the A tensor) [m_pool][2^n][2], and
 * validation states xv, yv = U xv [v][2^n][2] (v may be 0).  Host
 * pointers; copied.  Training set = the first M rows of the pool; doubling
 * takes the first 2M rows (prefix-nested, R13).  Rows should be orthonormal
 * Haar states; this is documented, not checked. */
qfs_status qfs_set_samples(qfs_ctx *c, int m_pool, const double *x, const double *y, int v,
                           const double *xv, const double *yv);

/* Asynchronous variant for pipelined callers: queues the sample set (same
 * arguments and layout as qfs_set_samples) into one of two device staging
 * slots with host->device copies on a separate copy stream, and returns at
 * once; the copies start behind the forward phase of the next sweep the
 * context runs (or at once if no sweep runs before the set is needed); the
 * next qfs_instantiate / qfs_trace_sweeps / qfs_bench_sweeps call
 * consumes the oldest queued set (finite check, transpose to the sample-minor
 * pools) before it runs.  So a caller can queue step t+1's samples while step
 * t's instantiation runs.  The host buffers must stay valid and unmodified
 * until the consuming call returns (pinned memory makes the copies overlap).
 * QFS_ERR_STATE when two sets are already queued; argument errors as
 * qfs_set_samples; a non-finite sample is reported (QFS_ERR_NUMERIC) by the
 * consuming call after its first sweep (the check rides on the initial-gate
 * check's read-back, no extra host round trip; outputs are not written and
 * the context has no samples until the next qfs_set_samples*). */
qfs_status qfs_set_samples_async(qfs_ctx *c, int m_pool, const double *x, const double *y, int v,
                                 const double *xv, const double *yv);

/* QFactor's full-unitary inputs without storing them (
 * with M = 2^n orthonormal inputs the sample cost is the full
 * Hilbert-Schmidt cost): training input m is the computational basis state
 * x_m = e_m (|m>, little-endian) for m < m_pool, generated inside the kernels
 * that read x (the first forward pass, gate 0's environment, the sweep-end
 * cost) — the 2^n x m_pool x pool is never stored or copied.  y [m_pool][2^n][2]
 * holds the targets y_m = U e_m (the columns of U; host, copied); validation as
 * qfs_set_samples.  Pair contexts on one rank only (QFS_ERR_ARG in sample mode,
 * for emulated ranks or block circuits); the sweep runs on the streamed path.
 * A later qfs_set_samples returns to stored inputs. */
qfs_status qfs_set_samples_basis(qfs_ctx *c, int m_pool, const double *y, int v, const double *xv,
                                 const double *yv);

/* Same, from DEVICE pointers (e.g. torch CUDA tensors) on cuda_stream
 * (cudaStream_t, NULL = legacy default stream).  Copies device-to-device. */
qfs_status qfs_set_samples_device(qfs_ctx *c, int m_pool, const void *dx, const void *dy, int v,
                                  const void *dxv, const void *dyv, void *cuda_stream);

/* Instantiate from s starts in lockstep (P:378 multistarts): init_gates host
 * [s][k][4][4][2]; out_gates host [s][k][4][4][2]; out host [s]; *winner = the
 * lowest-index start converged at the earliest converging sweep, else the
 * minimum c_train start (ties: lower index).  The initial gates are validated
 * on the device (finite; ||G^dag G - I||_max <= 1e-10; QFS_GATE_VAR1 slots of
 * the form u (x) I); a failure is reported as QFS_ERR_NUMERIC after the first
 * sweep, and then out_gates / out are not written.  Page-locked (pinned,
 * mapped) init_gates / out_gates buffers are read / written by the device in
 * place; pageable ones go through the context's pinned staging buffer.  Both
 * are owned by the caller and not retained after the call returns. */
qfs_status qfs_instantiate(qfs_ctx *c, int s, const double *init_gates, const qfs_params *p,
                           double *out_gates, qfs_result *out, int *winner);

/* Parity / debug: n_sweeps sweeps at fixed M for s starts, no controller.
 * Any trace pointer may be NULL.  Layouts (host):
 *   env_trace   [n_sweeps][k][s][4][4][2]  environment E_i of gate i in sweep t
 *   gate_trace  [n_sweeps][s][k][4][4][2]  gates after sweep t
 *   cost_trace  [n_sweeps][s]              c_train after sweep t
 *   sigma_trace [n_sweeps][k][s]           sum of singular values of E'_i */
qfs_status qfs_trace_sweeps(qfs_ctx *c, int s, const double *init_gates, int m, double beta,
                            int n_sweeps, double *env_trace, double *gate_trace,
                            double *cost_trace, double *sigma_trace);

/* Throughput: exactly n_sweeps sweeps at fixed M for all s starts (no
 * controller, no validation); *sec = elapsed seconds from CUDA events. */
qfs_status qfs_bench_sweeps(qfs_ctx *c, int s, const double *init_gates, int m, int n_sweeps,
                            double *sec);

/* Kernel-level entry points (unit tests of each kernel against the oracle).
 * All host pointers; each call copies in, runs ONE kernel launch, copies out. */
/* psi [m][2^n][2] in place: psi <- G psi (dagger: G^dag psi) on (p0, p1). */
qfs_status qfs_op_apply(qfs_ctx *c, int p0, int p1, const double *g, int dagger, int m,
                        double *psi);
/* env [4][4][2] = sum_m sum_r phi[idx(l_in)] conj(chi[idx(l_out)]). */
qfs_status qfs_op_environment(qfs_ctx *c, int p0, int p1, int m, const double *phi,
                              const double *chi, double *env);
/* batch polar update: g_new[i] = Y X^dag of SVD((1-beta) env[i] + beta g_old[i]^dag),
 * sigma_sum[i] = sum of singular values; env, g_old, g_new [count][4][4][2]. */
qfs_status qfs_op_polar(qfs_ctx *c, int count, const double *env, const double *g_old,
                        double beta, double *g_new, double *sigma_sum);

/* Profiling: when enabled, every kernel launch is bracketed by CUDA events on
 * the library's stream and accumulated per kernel class.  qfs_profile_read
 * fills up to cap entries: names (static strings), launches, total ms,
 * algorithmic bytes and flops; returns the number of classes in *count. */
qfs_status qfs_profile_enable(qfs_ctx *c, int on);
qfs_status qfs_profile_read(qfs_ctx *c, int cap, const char **names, long long *launches,
                            double *ms, double *bytes, double *flops, int *count);

/* Gate kinds ("possibly multi-qubit
 * unitary gates", Table 1's U3 + CNOT circuits; readings R24-R25).
 * Every slot is still a 4x4 block on its pair (p0, p1):
 *   QFS_GATE_VAR2  two-qubit variable unitary (default): G <- Y X^dag, E = X D Y^dag;
 *   QFS_GATE_FIXED constant gate (e.g. CNOT): applied, never updated; its sum
 *                  sigma slot reports Re Tr(E G);
 *   QFS_GATE_VAR1  one-qubit variable unitary u on p0, stored as u (x) I (p1 is a
 *                  carrier the block acts trivially on): u <- Y X^dag from the SVD
 *                  of E1[a][b] = E[a][b] + E[a+2][b+2] (Tr(E (u (x) I)) = Tr(E1 u)).
 * qfs_set_gate_kinds(c, kinds[k]) sets them (NULL: all QFS_GATE_VAR2);
 * QFS_ERR_ARG for another value.  Initial gates of QFS_GATE_VAR1 slots must be
 * of the form u (x) I (else qfs_instantiate / qfs_trace_sweeps return
 * QFS_ERR_NUMERIC); fixed slots take their constant from the initial gates. */
enum { QFS_GATE_VAR2 = 0, QFS_GATE_FIXED = 1, QFS_GATE_VAR1 = 2 };
qfs_status qfs_set_gate_kinds(qfs_ctx *c, const int32_t *kinds);

/* Sweep implementation: 0 = auto (default; cluster-resident
 * whenever a start's states fit in the shared memory of a cluster of <= 16
 * CTAs, else streamed), 1 = streamed (B cache in HBM, one fused launch per
 * gate), 2 = cluster-resident only (a sweep whose states do not fit fails with
 * QFS_ERR_CAPACITY).  Both compute the same sweep; the
 * resident one recovers B_i = G_i^dag B_{i+1} instead of storing the B cache
 * (P:165), which changes results only at rounding level.  QFS_ERR_ARG for
 * another value.  Takes effect at the next sweep. */
qfs_status qfs_set_path(qfs_ctx *c, int path);

/* Number of kernel launches issued since the context was created. */
long long qfs_launch_count(const qfs_ctx *c);
/* The library's CUDA stream (cudaStream_t) — for callers that order work. */
void *qfs_stream(const qfs_ctx *c);

const char *qfs_last_error(const qfs_ctx *c);
void qfs_destroy(qfs_ctx *c);

#ifdef __cplusplus
}
#endif
#endif
