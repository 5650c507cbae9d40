// qfso.cpp — CPU ORACLE for QFactor-Sample instantiation (arXiv 2405.12866).
//
// TEST INFRASTRUCTURE ONLY (see qfso.h).  Plain, slow, obviously correct:
// dense loops in double, long double accumulation, its own Jacobi SVD, no BLAS,
// no SIMD, no blocking or fusion beyond what the paper's algorithm states.
// OpenMP (if enabled) only runs independent multistarts side by side.
//
// Citations: P:<line> = /root/reference/PAPER.md line; DESIGN.md §2 lists the
// readings taken where the paper is silent (numbered R1..R21 there and below).
#include "qfso.h"

#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <limits>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

typedef std::complex<double> cd;
typedef std::complex<long double> cld;

// ---------------------------------------------------------------- indexing --
// R1: little-endian amplitudes; the quadruple r of a gate on (p0, p1) is the
// r-th assignment of the other n-2 qubits, obtained by inserting zero bits at
// the two gate positions (ascending); member l sits at base | b0<<p0 | b1<<p1
// with l = b0 + 2 b1.
inline long insert_zero_bit(long v, int pos) {
  long low = v & ((1L << pos) - 1);
  long high = v >> pos;
  return (high << (pos + 1)) | low;
}
inline long quad_base(long r, int p0, int p1) {
  int lo = p0 < p1 ? p0 : p1, hi = p0 < p1 ? p1 : p0;
  return insert_zero_bit(insert_zero_bit(r, lo), hi);
}
inline long quad_index(long base, int l, int p0, int p1) {
  return base | (long)(l & 1) << p0 | (long)((l >> 1) & 1) << p1;
}

inline cd ld(const double *p, long i) { return cd(p[2 * i], p[2 * i + 1]); }
inline void st(double *p, long i, cd v) { p[2 * i] = v.real(); p[2 * i + 1] = v.imag(); }

bool valid_pair(int n, int p0, int p1) {
  return n >= 2 && p0 >= 0 && p1 >= 0 && p0 < n && p1 < n && p0 != p1;
}

// ------------------------------------------------------------- gate apply --
// P:59 ("QFactor utilizes tensor network contractions"), P:127 (B tensors):
// psi[idx(l_out)] <- sum_l G[l_out][l] psi[idx(l)] for every quadruple.
void apply_gate(int n, int p0, int p1, const cd G[16], int m, double *psi) {
  const long N = 1L << n;
  for (int s = 0; s < m; ++s) {
    double *row = psi + 2 * (long)s * N;
    for (long r = 0; r < N / 4; ++r) {
      long base = quad_base(r, p0, p1);
      cd v[4];
      for (int l = 0; l < 4; ++l) v[l] = ld(row, quad_index(base, l, p0, p1));
      for (int lo = 0; lo < 4; ++lo) {
        cd acc = 0;
        for (int l = 0; l < 4; ++l) acc += G[4 * lo + l] * v[l];
        st(row, quad_index(base, lo, p0, p1), acc);
      }
    }
  }
}

void load_gate(const double *g, cd G[16]) {
  for (int i = 0; i < 16; ++i) G[i] = cd(g[2 * i], g[2 * i + 1]);
}
void adjoint(const cd A[16], cd Ad[16]) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) Ad[4 * i + j] = std::conj(A[4 * j + i]);
}

// ------------------------------------------------------------ environment --
// P:121-125 ("for any specific gate u_i ... can be written as Re(Tr(E u_i))"),
// P:172 (Fig. env_calc: trace all legs except the gate's): R4 orientation
// E[l_in][l_out] = sum_m sum_r phi_m[idx_r(l_in)] conj(chi_m[idx_r(l_out)]),
// so that Tr(E G) = sum_m <chi_m | G phi_m>.  Accumulated in long double in the
// order m ascending, then r ascending.
void environment(int n, int p0, int p1, int m0, int m1, int mstride, const double *phi,
                 const double *chi, cld E[16]) {
  const long N = 1L << n;
  for (int m = m0; m < m1; m += mstride) {
    const double *f = phi + 2 * (long)m * N;
    const double *c = chi + 2 * (long)m * N;
    for (long r = 0; r < N / 4; ++r) {
      long base = quad_base(r, p0, p1);
      cd fv[4], cv[4];
      for (int l = 0; l < 4; ++l) {
        fv[l] = ld(f, quad_index(base, l, p0, p1));
        cv[l] = ld(c, quad_index(base, l, p0, p1));
      }
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
          cd t = fv[a] * std::conj(cv[b]);
          E[4 * a + b] += cld(t.real(), t.imag());
        }
    }
  }
}

// ------------------------------------------------------------------- SVD --
// E = X D Y^dag, u_new = Y X^dag.  The paper does not name its SVD
// routine (R5); the oracle uses Hestenes one-sided Jacobi: complex rotations on
// column pairs (j, k) from the right, chosen so the new a_j^dag a_k = 0, and
// accumulated into V.  Converged when every pair has
// |a_j^dag a_k| <= 1e-15 ||a_j|| ||a_k|| (cap 30 sweeps).  Then
// sigma_j = ||a_j||, X_j = a_j / sigma_j, Y = V.  Columns with
// sigma_j <= 1e-14 sigma_max are numerically null: X_j is completed by
// Gram-Schmidt on e_0..e_3 against the other columns (R5).
// D x D (D = 4: two-qubit blocks; D = 2: one-qubit gates, reading R24), row-major.
template <int D>
int svd_jacobi(const cd *A_in, cd *X, double *sigma, cd *Y) {
  cd A[D * D], V[D * D];
  for (int i = 0; i < D * D; ++i) { A[i] = A_in[i]; V[i] = (i % (D + 1) == 0) ? cd(1, 0) : cd(0, 0); }
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    bool rotated = false;
    for (int j = 0; j < D - 1; ++j)
      for (int k = j + 1; k < D; ++k) {
        double alpha = 0, beta = 0;
        cd gamma = 0;
        for (int r = 0; r < D; ++r) {
          alpha += std::norm(A[D * r + j]);
          beta += std::norm(A[D * r + k]);
          gamma += std::conj(A[D * r + j]) * A[D * r + k];
        }
        double ag = std::abs(gamma);
        if (ag == 0.0 || ag <= 1e-15 * std::sqrt(alpha) * std::sqrt(beta)) continue;
        rotated = true;
        cd ph = gamma / ag;                       // e^{i phi}
        double zeta = (beta - alpha) / (2.0 * ag);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + t * t);
        double s = c * t;
        // [a_j' a_k'] = [a_j a_k] J,  J = [[c, s e^{i phi}], [-s e^{-i phi}, c]]
        for (int r = 0; r < D; ++r) {
          cd aj = A[D * r + j], ak = A[D * r + k];
          A[D * r + j] = c * aj - s * std::conj(ph) * ak;
          A[D * r + k] = s * ph * aj + c * ak;
          cd vj = V[D * r + j], vk = V[D * r + k];
          V[D * r + j] = c * vj - s * std::conj(ph) * vk;
          V[D * r + k] = s * ph * vj + c * vk;
        }
      }
    if (!rotated) break;
  }
  double smax = 0;
  for (int j = 0; j < D; ++j) {
    double nn = 0;
    for (int r = 0; r < D; ++r) nn += std::norm(A[D * r + j]);
    sigma[j] = std::sqrt(nn);
    if (sigma[j] > smax) smax = sigma[j];
  }
  bool null_col[D];
  for (int j = 0; j < D; ++j) {
    null_col[j] = !(sigma[j] > 1e-14 * smax) || smax == 0.0;
    for (int r = 0; r < D; ++r) X[D * r + j] = null_col[j] ? cd(0, 0) : A[D * r + j] / sigma[j];
  }
  // complete null columns: Gram-Schmidt of e_0..e_{D-1} against the filled columns
  for (int j = 0; j < D; ++j) {
    if (!null_col[j]) continue;
    for (int e = 0; e < D; ++e) {
      cd v[D];
      for (int r = 0; r < D; ++r) v[r] = (r == e) ? cd(1, 0) : cd(0, 0);
      for (int pass = 0; pass < 2; ++pass)
        for (int q = 0; q < D; ++q) {
          if (q == j || (null_col[q] && q > j)) continue;
          cd d = 0;
          for (int r = 0; r < D; ++r) d += std::conj(X[D * r + q]) * v[r];
          for (int r = 0; r < D; ++r) v[r] -= d * X[D * r + q];
        }
      double nv = 0;
      for (int r = 0; r < D; ++r) nv += std::norm(v[r]);
      nv = std::sqrt(nv);
      if (nv > 0.5) {
        for (int r = 0; r < D; ++r) X[D * r + j] = v[r] / nv;
        break;
      }
    }
  }
  for (int i = 0; i < D * D; ++i) Y[i] = V[i];
  return sweep;
}
int svd4(const cd A_in[16], cd X[16], double sigma[4], cd Y[16]) { return svd_jacobi<4>(A_in, X, sigma, Y); }

// P:59-62 with the beta term of P:380-386 (R15: u = the current, old gate):
// E' = (1 - beta) E + beta u^dag;  E' = X D Y^dag;  u_new = Y X^dag.
void polar_update(const cd E[16], const cd Gold[16], double beta, cd Gnew[16], double *sig_sum) {
  cd Ep[16], Gd[16], X[16], Y[16];
  double sg[4];
  adjoint(Gold, Gd);
  for (int i = 0; i < 16; ++i) Ep[i] = (1.0 - beta) * E[i] + beta * Gd[i];
  svd4(Ep, X, sg, Y);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      cd acc = 0;
      for (int j = 0; j < 4; ++j) acc += Y[4 * a + j] * std::conj(X[4 * b + j]);
      Gnew[4 * a + b] = acc;
    }
  if (sig_sum) *sig_sum = sg[0] + sg[1] + sg[2] + sg[3];
}

// Gate update by kind ("possibly multi-qubit
// unitary gates", Table 1's U3 + CNOT circuits; readings R24-R25):
//   kind 0 (two-qubit variable block): polar_update above;
//   kind 1 (fixed gate, e.g. CNOT): never updated; *sig_sum = Re Tr(E G);
//   kind 2 (one-qubit variable gate u on the pair's first qubit p0, stored as
//     the block G = u (x) I on (p0, p1), l = b(p0) + 2 b(p1)): since
//     Tr(E (u (x) I)) = Tr(E1 u) with E1[a][b] = sum_c E[a + 2c][b + 2c] (the
//     partial trace over the p1 bit), u_new = Y X^dag from the 2x2 SVD of
//     E1' = (1 - beta) E1 + beta u_old^dag, and G_new = u_new (x) I exactly.
enum { KIND_VAR2 = 0, KIND_FIXED = 1, KIND_VAR1 = 2 };

void gate_update(int kind, const cd E[16], const cd Gold[16], double beta, cd Gnew[16], double *sig_sum) {
  if (kind == KIND_FIXED) {
    cd tr = 0;
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) tr += E[4 * a + b] * Gold[4 * b + a];
    for (int i = 0; i < 16; ++i) Gnew[i] = Gold[i];
    if (sig_sum) *sig_sum = tr.real();
    return;
  }
  if (kind != KIND_VAR1) {
    polar_update(E, Gold, beta, Gnew, sig_sum);
    return;
  }
  cd E1[4], X[4], Y[4];
  double sg[2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const cd uo_dag = std::conj(Gold[4 * b + a]);  // u_old^dag[a][b] = conj(u_old[b][a])
      E1[2 * a + b] = (1.0 - beta) * (E[4 * a + b] + E[4 * (a + 2) + b + 2]) + beta * uo_dag;
    }
  svd_jacobi<2>(E1, X, sg, Y);
  cd u[4];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) u[2 * a + b] = Y[2 * a + 0] * std::conj(X[2 * b + 0]) + Y[2 * a + 1] * std::conj(X[2 * b + 1]);
  for (int lo = 0; lo < 4; ++lo)
    for (int li = 0; li < 4; ++li)
      Gnew[4 * lo + li] = ((lo >> 1) == (li >> 1)) ? u[2 * (lo & 1) + (li & 1)] : cd(0, 0);
  if (sig_sum) *sig_sum = sg[0] + sg[1];
}

// ------------------------------------------------------------------ cost --
// P:116-120 (eq:qfactor_sample_cost_function), direct form (R6):
// (1/M) sum_j ||a_j - b_j||^2, accumulated in long double.
long double sq_distance_sum(int n, int m0, int m1, int mstride, const double *a,
                            const double *b) {
  const long N = 1L << n;
  long double acc = 0;
  for (int m = m0; m < m1; m += mstride)
    for (long i = 0; i < N; ++i) {
      long double dr = (long double)a[2 * ((long)m * N + i)] - b[2 * ((long)m * N + i)];
      long double di = (long double)a[2 * ((long)m * N + i) + 1] - b[2 * ((long)m * N + i) + 1];
      acc += dr * dr + di * di;
    }
  return acc;
}

// ----------------------------------------------------------------- sweep --
// One sweep for one start ("sweeps the circuit from right to left";
// P:127/P:165 A and B tensors; P:172 Fig. env_calc; R2, R3):
//  (a) B_0 = x, B_{i} = G_{i-1} B_{i-1} (previous sweep's gates, gate 0 first)
//  (b) chi = y  (the A tensor, conjugated)
//  (c) for i = K-1 .. 0: E_i = env(B_i, chi); G_i <- polar(E_i); chi <- G_i^dag chi
//  (d) c_train = (1/M) sum ||chi - x||^2   (chi = C_new^dag y)
// g > 1: sample-shard emulation — E_i and the cost sum are formed per shard
// r (rows m = r mod g) and summed in rank order.
struct SweepOut {
  std::vector<cd> env;     // [K][16] (as seen, before the update)
  std::vector<double> sig; // [K]
  double c_train;
};

void sweep_one(int n, int K, const int32_t *pairs, const int32_t *kinds, cd *G /*[K][16] in/out*/, int M,
               const double *x, const double *y, double beta, int g, SweepOut *out,
               std::vector<double> &Bbuf, std::vector<double> &chi) {
  const long N = 1L << n;
  const long rowlen = 2 * (long)M * N;
  Bbuf.resize((size_t)K * rowlen);
  chi.resize(rowlen);
  std::memcpy(Bbuf.data(), x, sizeof(double) * rowlen);
  for (int i = 1; i < K; ++i) {
    double *Bi = Bbuf.data() + (size_t)i * rowlen;
    std::memcpy(Bi, Bbuf.data() + (size_t)(i - 1) * rowlen, sizeof(double) * rowlen);
    apply_gate(n, pairs[2 * (i - 1)], pairs[2 * (i - 1) + 1], G + 16 * (i - 1), M, Bi);
  }
  std::memcpy(chi.data(), y, sizeof(double) * rowlen);
  if (out) { out->env.assign((size_t)K * 16, cd(0, 0)); out->sig.assign(K, 0.0); }
  for (int i = K - 1; i >= 0; --i) {
    int p0 = pairs[2 * i], p1 = pairs[2 * i + 1];
    cld Etot[16];
    for (int q = 0; q < 16; ++q) Etot[q] = 0;
    for (int r = 0; r < g; ++r) {
      cld Er[16];
      for (int q = 0; q < 16; ++q) Er[q] = 0;
      environment(n, p0, p1, r, M, g, Bbuf.data() + (size_t)i * rowlen, chi.data(), Er);
      for (int q = 0; q < 16; ++q) Etot[q] += cd((double)Er[q].real(), (double)Er[q].imag());
    }
    cd E[16];
    for (int q = 0; q < 16; ++q) E[q] = cd((double)Etot[q].real(), (double)Etot[q].imag());
    cd Gn[16], Gd[16];
    double ss = 0;
    gate_update(kinds ? kinds[i] : KIND_VAR2, E, G + 16 * i, beta, Gn, &ss);
    for (int q = 0; q < 16; ++q) G[16 * i + q] = Gn[q];
    if (out) {
      for (int q = 0; q < 16; ++q) out->env[16 * i + q] = E[q];
      out->sig[i] = ss;
    }
    adjoint(Gn, Gd);
    apply_gate(n, p0, p1, Gd, M, chi.data());
  }
  long double tot = 0;
  for (int r = 0; r < g; ++r) tot += (double)sq_distance_sum(n, r, M, g, chi.data(), x);
  if (out) out->c_train = (double)(tot / (long double)M);
}

// c_val = (1/V) sum_v ||y_v - C x_v||^2 through all K gates G
// (the caller passes the post-sweep gates, R7).  Pinned against a dense U and C
// (tests/test_oracle_pins.py::test_validation_cost_dense_brute_force).
double validation_cost(int n, int K, const int32_t *pairs, const cd *G, int V, const double *xv,
                       const double *yv) {
  const long N = 1L << n;
  std::vector<double> psi(xv, xv + 2 * (long)V * N);
  for (int i = 0; i < K; ++i) apply_gate(n, pairs[2 * i], pairs[2 * i + 1], G + 16 * i, V, psi.data());
  return (double)(sq_distance_sum(n, 0, V, 1, psi.data(), yv) / (long double)V);
}

// ------------------------------------------------------------ blocks --
// Multi-qubit blocks (P:57 QFactor updates "possibly
// multi-qubit" unitary gates without parameterising them).  A block of arity
// a in {2, 3} acts on qubits q_0..q_{a-1} (as given) with the d x d matrix
// G[l_out][l_in], d = 2^a, local index l = sum_j b(q_j) 2^j (reading R1
// extended: the first listed qubit is the least significant local bit).
// Gates of a circuit are stored packed, gate k at complex offset off_k =
// sum_{j<k} d_j^2.  Everything below is the same algorithm as the pair code
// above with 4 replaced by d.
struct Block {
  int a;     // arity
  int q[3];  // qubits (q[2] unused for a = 2)
};
inline long blk_base(long r, const Block &b) {
  int srt[3] = {b.q[0], b.q[1], b.a > 2 ? b.q[2] : 0};
  for (int i = 0; i < b.a; ++i)
    for (int j = i + 1; j < b.a; ++j)
      if (srt[j] < srt[i]) { int t = srt[i]; srt[i] = srt[j]; srt[j] = t; }
  long v = r;
  for (int i = 0; i < b.a; ++i) v = insert_zero_bit(v, srt[i]);
  return v;
}
inline long blk_index(long base, int l, const Block &b) {
  long v = base;
  for (int j = 0; j < b.a; ++j) v |= (long)((l >> j) & 1) << b.q[j];
  return v;
}

void apply_block(int n, const Block &b, const cd *G, int m, double *psi) {
  const long N = 1L << n;
  const int d = 1 << b.a;
  for (int s = 0; s < m; ++s) {
    double *row = psi + 2 * (long)s * N;
    for (long r = 0; r < (N >> b.a); ++r) {
      long base = blk_base(r, b);
      cd v[8];
      for (int l = 0; l < d; ++l) v[l] = ld(row, blk_index(base, l, b));
      for (int lo = 0; lo < d; ++lo) {
        cd acc = 0;
        for (int l = 0; l < d; ++l) acc += G[d * lo + l] * v[l];
        st(row, blk_index(base, lo, b), acc);
      }
    }
  }
}

void adjoint_d(int d, const cd *A, cd *Ad) {
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) Ad[d * i + j] = std::conj(A[d * j + i]);
}

// E[l_in][l_out] = sum_m sum_r phi_m[idx_r(l_in)] conj(chi_m[idx_r(l_out)]) (R4)
void environment_block(int n, const Block &b, int m0, int m1, int mstride, const double *phi,
                       const double *chi, cld *E) {
  const long N = 1L << n;
  const int d = 1 << b.a;
  for (int m = m0; m < m1; m += mstride) {
    const double *f = phi + 2 * (long)m * N;
    const double *c = chi + 2 * (long)m * N;
    for (long r = 0; r < (N >> b.a); ++r) {
      long base = blk_base(r, b);
      cd fv[8], cv[8];
      for (int l = 0; l < d; ++l) {
        fv[l] = ld(f, blk_index(base, l, b));
        cv[l] = ld(c, blk_index(base, l, b));
      }
      for (int x = 0; x < d; ++x)
        for (int y = 0; y < d; ++y) {
          cd t = fv[x] * std::conj(cv[y]);
          E[d * x + y] += cld(t.real(), t.imag());
        }
    }
  }
}

// Gate update of a d x d block by kind: variable = Y X^dag from the SVD of
// E' = (1 - beta) E + beta G_old^dag; fixed = unchanged,
// *sig = Re Tr(E G); a two-qubit block keeps the kinds of gate_update (R24).
void gate_update_block(int kind, int d, const cd *E, const cd *Gold, double beta, cd *Gnew, double *sig) {
  if (d == 4) { gate_update(kind, E, Gold, beta, Gnew, sig); return; }
  if (kind == KIND_FIXED) {
    cd tr = 0;
    for (int a = 0; a < d; ++a)
      for (int c = 0; c < d; ++c) tr += E[d * a + c] * Gold[d * c + a];
    for (int i = 0; i < d * d; ++i) Gnew[i] = Gold[i];
    if (sig) *sig = tr.real();
    return;
  }
  cd Ep[64], Gd[64], X[64], Y[64];
  double sg[8];
  adjoint_d(d, Gold, Gd);
  for (int i = 0; i < d * d; ++i) Ep[i] = (1.0 - beta) * E[i] + beta * Gd[i];
  svd_jacobi<8>(Ep, X, sg, Y);
  for (int a = 0; a < d; ++a)
    for (int c = 0; c < d; ++c) {
      cd acc = 0;
      for (int j = 0; j < d; ++j) acc += Y[d * a + j] * std::conj(X[d * c + j]);
      Gnew[d * a + c] = acc;
    }
  double ss = 0;
  for (int j = 0; j < d; ++j) ss += sg[j];
  if (sig) *sig = ss;
}

struct BlockCircuit {
  int n, K, gsz;
  std::vector<Block> b;
  std::vector<int> off;  // [K + 1]
  const int32_t *kinds;
};

// one sweep of sweep_one's algorithm over blocks
void sweep_blocks(const BlockCircuit &C, cd *G /*packed, in/out*/, int M, const double *x,
                  const double *y, double beta, SweepOut *out, std::vector<double> &Bbuf,
                  std::vector<double> &chi) {
  const int n = C.n, K = C.K;
  const long N = 1L << n;
  const long rowlen = 2 * (long)M * N;
  Bbuf.resize((size_t)K * rowlen);
  chi.resize(rowlen);
  std::memcpy(Bbuf.data(), x, sizeof(double) * rowlen);
  for (int i = 1; i < K; ++i) {
    double *Bi = Bbuf.data() + (size_t)i * rowlen;
    std::memcpy(Bi, Bbuf.data() + (size_t)(i - 1) * rowlen, sizeof(double) * rowlen);
    apply_block(n, C.b[i - 1], G + C.off[i - 1], M, Bi);
  }
  std::memcpy(chi.data(), y, sizeof(double) * rowlen);
  if (out) { out->env.assign((size_t)C.gsz, cd(0, 0)); out->sig.assign(K, 0.0); }
  for (int i = K - 1; i >= 0; --i) {
    const int d = 1 << C.b[i].a;
    cld Et[64];
    for (int q = 0; q < d * d; ++q) Et[q] = 0;
    environment_block(n, C.b[i], 0, M, 1, Bbuf.data() + (size_t)i * rowlen, chi.data(), Et);
    cd E[64], Gn[64], Gd[64];
    for (int q = 0; q < d * d; ++q) E[q] = cd((double)Et[q].real(), (double)Et[q].imag());
    double ss = 0;
    gate_update_block(C.kinds ? C.kinds[i] : KIND_VAR2, d, E, G + C.off[i], beta, Gn, &ss);
    for (int q = 0; q < d * d; ++q) G[C.off[i] + q] = Gn[q];
    if (out) {
      for (int q = 0; q < d * d; ++q) out->env[C.off[i] + q] = E[q];
      out->sig[i] = ss;
    }
    adjoint_d(d, Gn, Gd);
    apply_block(n, C.b[i], Gd, M, chi.data());
  }
  if (out) out->c_train = (double)(sq_distance_sum(n, 0, M, 1, chi.data(), x) / (long double)M);
}

double validation_cost_blocks(const BlockCircuit &C, const cd *G, int V, const double *xv, const double *yv) {
  const long N = 1L << C.n;
  std::vector<double> psi(xv, xv + 2 * (long)V * N);
  for (int i = 0; i < C.K; ++i) apply_block(C.n, C.b[i], G + C.off[i], V, psi.data());
  return (double)(sq_distance_sum(C.n, 0, V, 1, psi.data(), yv) / (long double)V);
}

// structure check + packing offsets; kinds: 0 variable, 1 fixed, 2 one-qubit (arity 2 only)
int make_blocks(int n, int k, const int32_t *qubits, const int32_t *arity, const int32_t *kinds,
                BlockCircuit &C) {
  if (n < 2 || n > 30 || k < 1 || !qubits || !arity) return 1;
  C.n = n; C.K = k; C.kinds = kinds;
  C.b.resize(k);
  C.off.assign(k + 1, 0);
  for (int i = 0; i < k; ++i) {
    Block &b = C.b[i];
    b.a = arity[i];
    if (b.a != 2 && b.a != 3) return 1;
    for (int j = 0; j < 3; ++j) b.q[j] = qubits[3 * i + j];
    for (int j = 0; j < b.a; ++j) {
      if (b.q[j] < 0 || b.q[j] >= n) return 1;
      for (int t = 0; t < j; ++t)
        if (b.q[t] == b.q[j]) return 1;
    }
    if (kinds && (kinds[i] < 0 || kinds[i] > 2 || (kinds[i] == KIND_VAR1 && b.a != 2))) return 1;
    C.off[i + 1] = C.off[i] + (1 << (2 * b.a));
  }
  C.gsz = C.off[k];
  return 0;
}

int check_structure(int n, int k, const int32_t *pairs, const int32_t *kinds = nullptr) {
  if (n < 2 || n > 30 || k < 1 || !pairs) return 1;
  for (int i = 0; i < k; ++i) {
    if (!valid_pair(n, pairs[2 * i], pairs[2 * i + 1])) return 1;
    if (kinds && (kinds[i] < 0 || kinds[i] > 2)) return 1;
  }
  return 0;
}

// The controller, shared by the pair and block circuits: sweep(G, M, out, B, chi)
// runs one sweep of one start, val(G) its validation cost; gsz = complex
// entries of one start's gates.
template <class SweepFn, class ValFn>
int run_controller(long N, int gsz, int m_pool, int v, int s, const double *init_gates, const qfso_params *p,
                   double *out_gates, qfso_result *out, int *winner, int n_threads, SweepFn sweep, ValFn val) {
  struct St {
    std::vector<cd> G;
    int M, it, total, fails, restarts, term, conv_sweep;
    bool has_prev, active;
    double c_prev, c_train, c_val;
    std::vector<double> B, chi;
  };
  std::vector<St> S(s);
  for (int st = 0; st < s; ++st) {
    S[st].G.resize((size_t)gsz);
    for (int i = 0; i < gsz; ++i)
      S[st].G[i] = cd(init_gates[2 * ((size_t)st * gsz + i)], init_gates[2 * ((size_t)st * gsz + i) + 1]);
    S[st].M = p->m_init; S[st].it = 0; S[st].total = 0; S[st].fails = 0; S[st].restarts = 0;
    S[st].term = -1; S[st].conv_sweep = -1; S[st].has_prev = false; S[st].active = true;
    S[st].c_prev = 0; S[st].c_train = NAN; S[st].c_val = NAN;
  }
  const double otr = p->overtrain_ratio;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
  for (int t = 1;; ++t) {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int st = 0; st < s; ++st) {
      St &A = S[st];
      if (!A.active) continue;
      SweepOut so;
      sweep(A.G.data(), A.M, &so, A.B, A.chi);  // step 1
      A.c_train = so.c_train;
      A.c_val = v > 0 ? val(A.G.data()) : NAN;
    }
    bool any_conv = false;
    for (int st = 0; st < s; ++st) {
      St &A = S[st];
      if (!A.active) continue;
      A.it += 1; A.total += 1;
      const double c = A.c_train;
      const bool gen_check = v > 0 && std::isfinite(otr) && A.M < N;           // step 2
      bool conv = false;                                                       // step 3
      if (c <= p->dist_tol) {
        if (!gen_check) conv = true;
        else if (c < 1e-14) conv = A.c_val <= (1.0 + otr) * p->dist_tol;
        else conv = A.c_val / c - 1.0 <= otr;
      }
      if (conv) {
        A.term = 0; A.active = false; A.conv_sweep = t; any_conv = true;
        continue;
      }
      if (gen_check && A.it >= p->min_iter && A.c_val / c - 1.0 > otr) {       // step 4
        if (2 * A.M > m_pool && A.M < N) { A.term = 3; A.active = false; continue; }
        A.M = (int)std::min<long>(2L * A.M, N);
        A.it = 0; A.fails = 0; A.has_prev = false; A.restarts += 1;
      } else if (p->plateau_window > 0) {                                      // step 5
        if (A.has_prev)
          A.fails = (std::fabs(A.c_prev) - std::fabs(c) > p->diff_tol_r * std::fabs(c)) ? 0 : A.fails + 1;
        A.c_prev = c; A.has_prev = true;
        if (A.it >= p->min_iter && A.fails >= p->plateau_window) { A.term = 1; A.active = false; continue; }
      }
      if (A.total >= p->max_iter) { A.term = 2; A.active = false; }            // step 6
    }
    bool any_active = false;
    for (int st = 0; st < s; ++st) any_active |= S[st].active;
    if (any_conv && p->stop_on_first) {
      for (int st = 0; st < s; ++st)
        if (S[st].active) { S[st].active = false; S[st].term = 4; }
      any_active = false;
    }
    if (!any_active) break;
  }
  // winner: lowest index among the earliest converged;
  // else min c_train, ties to the lower index.
  int win = -1, best_sweep = 1 << 30;
  for (int st = 0; st < s; ++st)
    if (S[st].term == 0 && S[st].conv_sweep < best_sweep) { best_sweep = S[st].conv_sweep; win = st; }
  if (win < 0) {
    double best = INFINITY;
    for (int st = 0; st < s; ++st)
      if (S[st].c_train < best) { best = S[st].c_train; win = st; }
    if (win < 0) win = 0;
  }
  for (int st = 0; st < s; ++st) {
    for (int i = 0; i < gsz; ++i) {
      out_gates[2 * ((size_t)st * gsz + i)] = S[st].G[i].real();
      out_gates[2 * ((size_t)st * gsz + i) + 1] = S[st].G[i].imag();
    }
    out[st].c_train = S[st].c_train; out[st].c_val = S[st].c_val;
    out[st].sweeps = S[st].total; out[st].restarts = S[st].restarts;
    out[st].final_m = S[st].M; out[st].term = S[st].term;
  }
  if (winner) *winner = win;
  return 0;
}

}  // namespace

// ===================================================================== ABI ==
extern "C" {

int qfso_apply_gate(int n, int p0, int p1, const double *g, int dagger, int m, double *psi) {
  if (!valid_pair(n, p0, p1) || !g || !psi || m < 0) return 1;
  cd G[16], Gd[16];
  load_gate(g, G);
  if (dagger) { adjoint(G, Gd); apply_gate(n, p0, p1, Gd, m, psi); }
  else apply_gate(n, p0, p1, G, m, psi);
  return 0;
}

int qfso_circuit_forward(int n, int k, const int32_t *pairs, const double *gates, int m,
                         double *psi) {
  if (check_structure(n, k, pairs) || !gates || !psi) return 1;
  for (int i = 0; i < k; ++i) {
    cd G[16];
    load_gate(gates + 32 * i, G);
    apply_gate(n, pairs[2 * i], pairs[2 * i + 1], G, m, psi);
  }
  return 0;
}

int qfso_environment(int n, int p0, int p1, int m, const double *phi, const double *chi,
                     double *env) {
  if (!valid_pair(n, p0, p1) || !phi || !chi || !env || m < 0) return 1;
  cld E[16];
  for (int q = 0; q < 16; ++q) E[q] = 0;
  environment(n, p0, p1, 0, m, 1, phi, chi, E);
  for (int q = 0; q < 16; ++q) { env[2 * q] = (double)E[q].real(); env[2 * q + 1] = (double)E[q].imag(); }
  return 0;
}

int qfso_svd4(const double *a, double *x, double *sigma, double *y, int *sweeps) {
  if (!a || !x || !sigma || !y) return 1;
  cd A[16], X[16], Y[16];
  load_gate(a, A);
  int sw = svd4(A, X, sigma, Y);
  for (int i = 0; i < 16; ++i) {
    x[2 * i] = X[i].real(); x[2 * i + 1] = X[i].imag();
    y[2 * i] = Y[i].real(); y[2 * i + 1] = Y[i].imag();
  }
  if (sweeps) *sweeps = sw;
  return 0;
}

int qfso_polar_update(const double *env, const double *g_old, double beta, double *g_new,
                      double *sigma_sum) {
  if (!env || !g_old || !g_new) return 1;
  cd E[16], Go[16], Gn[16];
  load_gate(env, E);
  load_gate(g_old, Go);
  polar_update(E, Go, beta, Gn, sigma_sum);
  for (int i = 0; i < 16; ++i) { g_new[2 * i] = Gn[i].real(); g_new[2 * i + 1] = Gn[i].imag(); }
  return 0;
}

// Scaled Newton iteration for the unitary polar factor (self-check of svd4):
// W <- (zeta W + (zeta W)^{-dag}) / 2, zeta = sqrt(||W^{-1}||_F / ||W||_F).
int qfso_newton_polar(const double *a, double *w, int *iters) {
  if (!a || !w) return 1;
  cd W[16];
  load_gate(a, W);
  int it = 0;
  for (; it < 100; ++it) {
    // inverse by Gauss-Jordan with partial pivoting
    cd M[4][8];
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 8; ++c) M[r][c] = c < 4 ? W[4 * r + c] : (c - 4 == r ? cd(1, 0) : cd(0, 0));
    for (int c = 0; c < 4; ++c) {
      int piv = c;
      for (int r = c + 1; r < 4; ++r) if (std::abs(M[r][c]) > std::abs(M[piv][c])) piv = r;
      if (std::abs(M[piv][c]) == 0.0) return 2;
      for (int q = 0; q < 8; ++q) std::swap(M[c][q], M[piv][q]);
      cd inv = 1.0 / M[c][c];
      for (int q = 0; q < 8; ++q) M[c][q] *= inv;
      for (int r = 0; r < 4; ++r) {
        if (r == c) continue;
        cd f = M[r][c];
        for (int q = 0; q < 8; ++q) M[r][q] -= f * M[c][q];
      }
    }
    double nw = 0, ni = 0;
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c) { nw += std::norm(W[4 * r + c]); ni += std::norm(M[r][c + 4]); }
    double zeta = std::sqrt(std::sqrt(ni) / std::sqrt(nw));
    cd Wn[16];
    double diff = 0, nn = 0;
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c) {
        // (W^{-1})^dag [r][c] = conj(Winv[c][r])
        Wn[4 * r + c] = 0.5 * (zeta * W[4 * r + c] + std::conj(M[c][r + 4]) / zeta);
        diff += std::norm(Wn[4 * r + c] - W[4 * r + c]);
        nn += std::norm(Wn[4 * r + c]);
      }
    for (int i = 0; i < 16; ++i) W[i] = Wn[i];
    if (std::sqrt(diff) <= 1e-15 * std::sqrt(nn)) { ++it; break; }
  }
  for (int i = 0; i < 16; ++i) { w[2 * i] = W[i].real(); w[2 * i + 1] = W[i].imag(); }
  if (iters) *iters = it;
  return 0;
}

double qfso_distance(int n, int m, const double *a, const double *b) {
  if (m <= 0) return 0.0;
  return (double)(sq_distance_sum(n, 0, m, 1, a, b) / (long double)m);
}

int qfso_trace_sweeps(int n, int k, const int32_t *pairs, int s, const double *init_gates, int m,
                      const double *x, const double *y, double beta, int n_sweeps, int g,
                      double *env_trace, double *gate_trace, double *cost_trace,
                      double *sigma_trace, int n_threads) {
  return qfso_trace_sweeps_kinds(n, k, pairs, nullptr, s, init_gates, m, x, y, beta, n_sweeps, g,
                                 env_trace, gate_trace, cost_trace, sigma_trace, n_threads);
}

int qfso_trace_sweeps_kinds(int n, int k, const int32_t *pairs, const int32_t *kinds, int s,
                            const double *init_gates, int m, const double *x, const double *y,
                            double beta, int n_sweeps, int g, double *env_trace, double *gate_trace,
                            double *cost_trace, double *sigma_trace, int n_threads) {
  if (check_structure(n, k, pairs, kinds) || s < 1 || m < 1 || m > (1 << n) || !init_gates || !x ||
      !y || n_sweeps < 0 || g < 1)
    return 1;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int st = 0; st < s; ++st) {
    std::vector<cd> G((size_t)k * 16);
    for (int i = 0; i < 16 * k; ++i)
      G[i] = cd(init_gates[2 * ((size_t)st * k * 16 + i)], init_gates[2 * ((size_t)st * k * 16 + i) + 1]);
    std::vector<double> B, chi;
    SweepOut so;
    for (int t = 0; t < n_sweeps; ++t) {
      sweep_one(n, k, pairs, kinds, G.data(), m, x, y, beta, g, &so, B, chi);
      if (env_trace)
        for (int i = 0; i < k; ++i)
          for (int q = 0; q < 16; ++q) {
            size_t o = ((((size_t)t * k + i) * s + st) * 16 + q) * 2;
            env_trace[o] = so.env[16 * i + q].real();
            env_trace[o + 1] = so.env[16 * i + q].imag();
          }
      if (gate_trace)
        for (int i = 0; i < 16 * k; ++i) {
          size_t o = (((size_t)t * s + st) * k * 16 + i) * 2;
          gate_trace[o] = G[i].real();
          gate_trace[o + 1] = G[i].imag();
        }
      if (cost_trace) cost_trace[(size_t)t * s + st] = so.c_train;
      if (sigma_trace)
        for (int i = 0; i < k; ++i) sigma_trace[((size_t)t * k + i) * s + st] = so.sig[i];
    }
  }
  return 0;
}

// Controller (P:114 double-and-restart, P:176 plateau
// window, P:182-192 generalisation check, P:354 keep gates on restart,
// P:360-378 hyperparameters; readings R7-R14, R16).
int qfso_instantiate(int n, int k, const int32_t *pairs, int m_pool, const double *x,
                     const double *y, int v, const double *xv, const double *yv, int s,
                     const double *init_gates, const qfso_params *p, double *out_gates,
                     qfso_result *out, int *winner, int n_threads) {
  return qfso_instantiate_kinds(n, k, pairs, nullptr, m_pool, x, y, v, xv, yv, s, init_gates, p,
                                out_gates, out, winner, n_threads);
}

int qfso_instantiate_kinds(int n, int k, const int32_t *pairs, const int32_t *kinds, int m_pool,
                           const double *x, const double *y, int v, const double *xv,
                           const double *yv, int s, const double *init_gates, const qfso_params *p,
                           double *out_gates, qfso_result *out, int *winner, int n_threads) {
  const long N = 1L << n;
  if (check_structure(n, k, pairs, kinds) || s < 1 || !p || !init_gates || !x || !y || !out_gates ||
      !out || m_pool < 1 || m_pool > N || p->m_init < 1 || p->m_init > m_pool || v < 0 ||
      (v > 0 && (!xv || !yv)) || p->max_iter < 1)
    return 1;
  return run_controller(
      N, 16 * k, m_pool, v, s, init_gates, p, out_gates, out, winner, n_threads,
      [&](cd *G, int M, SweepOut *so, std::vector<double> &B, std::vector<double> &chi) {
        sweep_one(n, k, pairs, kinds, G, M, x, y, p->beta, 1, so, B, chi);
      },
      [&](const cd *G) { return validation_cost(n, k, pairs, G, v, xv, yv); });
}

int qfso_bench_sweeps(int n, int k, const int32_t *pairs, int s, const double *init_gates, int m,
                      const double *x, const double *y, int n_sweeps, int n_threads,
                      double *sec) {
  auto t0 = std::chrono::steady_clock::now();
  int rc = qfso_trace_sweeps(n, k, pairs, s, init_gates, m, x, y, 0.0, n_sweeps, 1, nullptr,
                             nullptr, nullptr, nullptr, n_threads);
  auto t1 = std::chrono::steady_clock::now();
  if (sec) *sec = std::chrono::duration<double>(t1 - t0).count();
  return rc;
}

// ---------------------------------------------------------------- blocks --
int qfso_apply_block(int n, int arity, const int32_t *q, const double *g, int dagger, int m, double *psi) {
  const int32_t ar[1] = {arity};
  BlockCircuit C;
  if (!q || !g || !psi || m < 0 || make_blocks(n, 1, q, ar, nullptr, C)) return 1;
  const int d = 1 << arity;
  cd G[64], Gd[64];
  for (int i = 0; i < d * d; ++i) G[i] = cd(g[2 * i], g[2 * i + 1]);
  if (dagger) { adjoint_d(d, G, Gd); apply_block(n, C.b[0], Gd, m, psi); }
  else apply_block(n, C.b[0], G, m, psi);
  return 0;
}

int qfso_environment_block(int n, int arity, const int32_t *q, int m, const double *phi,
                           const double *chi, double *env) {
  const int32_t ar[1] = {arity};
  BlockCircuit C;
  if (!q || !phi || !chi || !env || m < 0 || make_blocks(n, 1, q, ar, nullptr, C)) return 1;
  const int d = 1 << arity;
  cld E[64];
  for (int i = 0; i < d * d; ++i) E[i] = 0;
  environment_block(n, C.b[0], 0, m, 1, phi, chi, E);
  for (int i = 0; i < d * d; ++i) { env[2 * i] = (double)E[i].real(); env[2 * i + 1] = (double)E[i].imag(); }
  return 0;
}

int qfso_polar_update_block(int d, const double *env, const double *g_old, double beta, double *g_new,
                            double *sigma_sum) {
  if ((d != 4 && d != 8) || !env || !g_old || !g_new) return 1;
  cd E[64], Go[64], Gn[64];
  for (int i = 0; i < d * d; ++i) { E[i] = cd(env[2 * i], env[2 * i + 1]); Go[i] = cd(g_old[2 * i], g_old[2 * i + 1]); }
  gate_update_block(KIND_VAR2, d, E, Go, beta, Gn, sigma_sum);
  for (int i = 0; i < d * d; ++i) { g_new[2 * i] = Gn[i].real(); g_new[2 * i + 1] = Gn[i].imag(); }
  return 0;
}

int qfso_trace_sweeps_blocks(int n, int k, const int32_t *qubits, const int32_t *arity, const int32_t *kinds,
                             int s, const double *init_gates, int m, const double *x, const double *y,
                             double beta, int n_sweeps, double *env_trace, double *gate_trace,
                             double *cost_trace, double *sigma_trace, int n_threads) {
  BlockCircuit C;
  if (make_blocks(n, k, qubits, arity, kinds, C) || s < 1 || m < 1 || m > (1 << n) || !init_gates || !x ||
      !y || n_sweeps < 0)
    return 1;
  const size_t gsz = (size_t)C.gsz;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int st = 0; st < s; ++st) {
    std::vector<cd> G(gsz);
    for (size_t i = 0; i < gsz; ++i)
      G[i] = cd(init_gates[2 * ((size_t)st * gsz + i)], init_gates[2 * ((size_t)st * gsz + i) + 1]);
    std::vector<double> B, chi;
    SweepOut so;
    for (int t = 0; t < n_sweeps; ++t) {
      sweep_blocks(C, G.data(), m, x, y, beta, &so, B, chi);
      if (env_trace)  // [t][gate-major: gate i at s * off_i, then start, then d_i^2 entries]
        for (int i = 0; i < k; ++i) {
          const int dd = C.off[i + 1] - C.off[i];
          for (int q = 0; q < dd; ++q) {
            size_t o = ((size_t)t * s * gsz + (size_t)s * C.off[i] + (size_t)st * dd + q) * 2;
            env_trace[o] = so.env[C.off[i] + q].real();
            env_trace[o + 1] = so.env[C.off[i] + q].imag();
          }
        }
      if (gate_trace)
        for (size_t i = 0; i < gsz; ++i) {
          size_t o = (((size_t)t * s + st) * gsz + i) * 2;
          gate_trace[o] = G[i].real();
          gate_trace[o + 1] = G[i].imag();
        }
      if (cost_trace) cost_trace[(size_t)t * s + st] = so.c_train;
      if (sigma_trace)
        for (int i = 0; i < k; ++i) sigma_trace[((size_t)t * k + i) * s + st] = so.sig[i];
    }
  }
  return 0;
}

int qfso_instantiate_blocks(int n, int k, const int32_t *qubits, const int32_t *arity, const int32_t *kinds,
                            int m_pool, const double *x, const double *y, int v, const double *xv,
                            const double *yv, int s, const double *init_gates, const qfso_params *p,
                            double *out_gates, qfso_result *out, int *winner, int n_threads) {
  const long N = 1L << n;
  BlockCircuit C;
  if (make_blocks(n, k, qubits, arity, kinds, C) || s < 1 || !p || !init_gates || !x || !y || !out_gates ||
      !out || m_pool < 1 || m_pool > N || p->m_init < 1 || p->m_init > m_pool || v < 0 ||
      (v > 0 && (!xv || !yv)) || p->max_iter < 1)
    return 1;
  return run_controller(
      N, C.gsz, m_pool, v, s, init_gates, p, out_gates, out, winner, n_threads,
      [&](cd *G, int M, SweepOut *so, std::vector<double> &B, std::vector<double> &chi) {
        sweep_blocks(C, G, M, x, y, p->beta, so, B, chi);
      },
      [&](const cd *G) { return validation_cost_blocks(C, G, v, xv, yv); });
}

}  // extern "C"
