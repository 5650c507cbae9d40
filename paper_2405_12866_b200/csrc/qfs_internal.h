// qfs_internal.h — launch-parameter structs shared by the runtime
// (qfs_runtime.cu) and the kernels (qfs_kernels.cu).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qfs {

// One active multistart in a lockstep launch: start index and its current
// number of (local) training rows.
struct Slot {
  int s;
  int m;
};

// Row addressing: row (s, m) of a state array starts at
//   base + (s * stride_s + m) * 2^n     (double2 elements)
// stride_s = 0 for the shared pools (x, y, xv, yv), M_cap for per-start buffers.
struct Rows {
  const double2 *base;
  long long stride_s;
};
struct RowsW {
  double2 *base;
  long long stride_s;
};

// Fused backward step for gate i (bwd_kernel):
//   chi <- G_{i+1}^dag chi (if update) and E_i += phi_i (x) conj(chi)
// over the 2^nu-amplitude groups spanned by the union of both gates' bits.
struct BwdParams {
  int n, nu, nb;              // qubits, union bits, blocks per start
  int upd_gate, env_gate;     // i+1 (or -1), i
  int K;
  const Slot *slots;
  Rows chi_src;
  RowsW chi_dst;              // base == nullptr: do not write chi back
  Rows phi;
  uint32_t ins[4];            // union bit positions, ascending (for zero insertion)
  long long off[16];          // amplitude offset of local index v (local bit t <-> loc[t])
  const double2 *gates;       // [S][K][16]
  double2 *gates_w;           // same array (written by the polar step)
  double *partials;           // [S_act][nb][32]
  unsigned *counters;         // [S_act]
  double *e_red;              // [S_act][32]: reduced E (sample mode: before all-reduce)
  int fuse_polar;             // 1: the last block of each start runs the polar update
  double beta;
  double *sig;                // [S][K] sum sigma, or nullptr
  double2 *env_trace;         // [K][S][16] for this sweep, or nullptr
  int S;                      // total starts (trace layout)
};

// Polar update of E (already reduced / all-reduced) for each active start.
struct PolarParams {
  int K, gate, S, n_slots;
  const Slot *slots;
  const double *e_red;        // [S_act][32]
  double2 *gates;             // [S][K][16]
  double beta;
  double *sig;                // [S][K] or nullptr
  double2 *env_trace;         // [K][S][16] or nullptr
};

// Sweep-end cost: chi' = G_0^dag chi ; sum_m ||chi'_m - x_m||^2 (direct form)
struct FinalParams {
  int n, nb;
  const Slot *slots;
  Rows chi;
  Rows x;
  int p0, p1;
  const double2 *gates;       // gate 0 of each start: gates + s*K*16
  int K;
  double *partials;           // [S_act][nb]
  unsigned *counters;         // [S_act]
  double *out_sum;            // [S_act] raw sum (host divides by M)
};

// Whole-row forward in shared memory (n <= 13): one CTA per (start, row).
//   mode 0 (train): writes B_1..B_{K-1} (B_{k+1} = G_k B_k, B_0 = x)
//   mode 1 (valid): applies all K gates, then sum ||row - yv_row||^2
struct FwdRowParams {
  int n, K, mode, rows;       // rows: number of validation rows (mode 1)
  const Slot *slots;
  const int2 *pairs;          // [K]
  const double2 *gates;       // [S][K][16]
  Rows src;                   // x pool / xv pool
  double2 *B;                 // mode 0: [K-1][S][M_cap][N]
  long long b_gate_stride;    // S * M_cap * N
  long long b_stride_s;       // M_cap
  Rows ref;                   // mode 1: yv pool
  double *row_out;            // mode 1: [S_act][rows] per-row sums
};

// Per-gate streamed forward (n >= 14): dst = G_k src for every row of every slot.
struct FwdGateParams {
  int n, nb, k, K, rows_fixed; // rows_fixed > 0: that many rows per start (validation)
  const Slot *slots;
  int p0, p1;
  const double2 *gates;
  Rows src;
  RowsW dst;
};

// Row distance sums (streamed validation end): out[j*rows + r] = ||a - b||^2
struct DistParams {
  int n, rows;
  const Slot *slots;
  Rows a, b;
  double *row_out;
};

// kernel-level unit ops
struct ApplyParams {
  int n, p0, p1, m;
  double2 g[16];              // already adjointed if requested
  double2 *psi;
};

// ---- launchers (qfs_kernels.cu); all return cudaGetLastError() ----
cudaError_t launch_bwd(const BwdParams &p, int n_slots, int tp0, int tp1, bool upd,
                       cudaStream_t st);
cudaError_t launch_polar(const PolarParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_final(const FinalParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_fwd_row(const FwdRowParams &p, int n_slots, int max_rows, cudaStream_t st);
cudaError_t launch_fwd_gate(const FwdGateParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_dist(const DistParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_row_reduce(const double *row_in, int rows, double *out, int n_slots,
                              cudaStream_t st);
cudaError_t launch_apply(const ApplyParams &p, cudaStream_t st);
cudaError_t launch_polar_batch(const double2 *env, const double2 *g_old, double beta,
                               double2 *g_new, double *sig, int count, cudaStream_t st);
int fwd_row_max_n();   // largest n the shared-memory row forward supports
int bwd_threads();

}  // namespace qfs
