// tables.hpp — setup-time FP64 construction of the translation tables the device kernels consume.
//
// The reference applies every translation (M2M, M2L, L2L) as a dense (P+1)^2 x (P+1)^2 complex
// matrix built from a Gaunt table (src/expansion.cpp:47-139).  The device path applies the SAME
// truncated operator factored as  T(t) = R(t^)^H · C(k|t|) · R(t^)
//   R : rotation taking t^ to +z; block-diagonal in n, real Wigner-d blocks times e^{im phi}
//   C : coaxial translation along +z; diagonal in m
// (O(P^3) instead of O(P^4) work per pair; identical under truncation because R does not mix
// degrees).  C is generated from the reference's own coupling formula specialised to t^ = z
// (expansion.cpp:111-122 with Y_lambda^{m-mu}(z^) = delta_{m,mu} sqrt((2 lambda+1)/4 pi)).
//
// FP32 range: device expansions are stored SCALED per tree level,
//   Mhat_n^m = M_n^m (2n+1)!! / s^n ,   Lhat_n^m = L_n^m s^n / (2n-1)!! ,   s = k * side(level),
// which keeps every stored number O(1) in the low-frequency regime the kd gate enforces.  The
// scale factors are folded into C here, in long double, so the kernels never see h_n or j_n.
#pragma once

#include <cstdint>
#include <vector>

#ifdef __CUDACC__
#define HFMM_HD __host__ __device__
#else
#define HFMM_HD
#endif

namespace hfmm_b200 {

// ---- FP64 special functions (own implementations; checked against the reference in tests) ----
void sph_jn_ld(int nmax, long double z, long double* out);               // j_0..j_nmax
void sph_hn_scaled(int nmax, double z, double* re, double* im);          // h_n z^{n+1}/(2n-1)!!
double wigner3j(int j1, int j2, int j3, int m1, int m2, int m3);
// Wigner small-d d^n_{mp,m}(beta), beta in [0, pi] given by cos(beta)
double wigner_d(int n, int mp, int m, double cos_beta);
long double double_factorial(int n);  // n!! for odd n >= -1

// Table layouts are padded so the device can fetch 4 rotation coefficients (or 2 complex coaxial
// coefficients) with one aligned 16-byte load; padding entries are zero.
//
// Rotation tables are stored FOLDED.  With xt_{-m} = (-1)^m x_{-m} the symmetry
// d^n_{-a,-b} = (-1)^{a-b} d^n_{a,b} splits a (2n+1)x(2n+1) block into
//   plus  system, size n+1 : inputs  [x_0, s_1..s_n],  s_m = x_m + xt_{-m}
//   minus system, size n   : inputs  [t_1..t_n],       t_m = x_m - xt_{-m}
// whose outputs are the same combinations of the rotated vector — half the multiply-adds.  The
// coaxial step acts identically on +m and -m, so it commutes with the folding and the whole
// pipeline (rotate, translate, rotate back) runs on folded vectors; they are folded once when the
// sources are gathered and unfolded once before the results are accumulated.
//   block n : plus  (n+1) rows of rot_plus_stride(n)  floats, entry [k][r] = input k -> output r
//             minus  n     rows of rot_minus_stride(n) floats, entry [k-1][r-1]
// Folded vector layout of degree n (same 2n+1 slots): n^2 + 0 : x_0 | n^2 + m : s_m | n^2 + n + m : t_m
HFMM_HD constexpr int rot_plus_stride(int n) { return (n + 1 + 3) & ~3; }
HFMM_HD constexpr int rot_minus_stride(int n) { return (n + 3) & ~3; }
HFMM_HD constexpr int rot_block_size(int n) {
  return (n + 1) * rot_plus_stride(n) + n * rot_minus_stride(n);
}
HFMM_HD constexpr int rot_block_offset(int n) {
  int off = 0;
  for (int j = 0; j < n; ++j) off += rot_block_size(j);
  return off;
}
HFMM_HD constexpr int rot_minus_offset(int n) { return rot_block_offset(n) + (n + 1) * rot_plus_stride(n); }
HFMM_HD constexpr int rot_table_size(int p) { return rot_block_offset(p + 1); }
HFMM_HD constexpr int coax_row_stride(int p, int m) { return (p + 1 - m + 1) & ~1; }
HFMM_HD constexpr int coax_block_offset(int p, int m) {
  int off = 0;
  for (int j = 0; j < m; ++j) off += (p + 1 - j) * coax_row_stride(p, j);
  return off;
}
HFMM_HD constexpr int coax_table_size(int p) { return coax_block_offset(p, p + 1); }  // complex

// Folded forward-rotation table for polar angle theta (layout above).  Unfolded, the forward
// rotation is  M'_n^{m'} = sum_m d^n_{m,m'}(theta) e^{i m phi} M_n^m ; the inverse rotation uses the
// same table through d^n_{mu,m'} = (-1)^{mu-m'} d^n_{m',mu}.
void build_rotation_table(int order, double cos_theta, float* out);
// the unfolded (2n+1)x(2n+1) block E_n[m][m'] = d^n_{m,m'} reconstructed from a folded table
// (row-major, index (m+n)*(2n+1) + (m'+n)); used by the CPU-side table tests
void unfold_rotation_block(int n, const float* folded_table, double* out);

enum class CoaxKind { m2l, m2m, l2l };
// Scaled coaxial coefficients Chat^m[n][nu] (complex, interleaved) for translation distance
// `dist` along +z at wavenumber k;  s_src / s_dst are the level scales of the source-side and
// destination-side expansions.
class CoaxBuilder {
 public:
  explicit CoaxBuilder(int order);
  // the builder of an order, constructed once per process (its 3j products depend on the order only)
  static const CoaxBuilder& shared(int order);
  // k + i k_imag: the (complex) wavenumber; the level scales s_src / s_dst are Re(k) * side
  void build(CoaxKind kind, double k, double dist, double s_src, double s_dst, float* out,
             double k_imag = 0.0) const;
  int order() const { return order_; }

 private:
  int order_;
  // A[m][nu][n][lambda slot]: real coupling (-1)^{(nu+lam-n)/2} (-1)^m (2lam+1)
  //   sqrt((2nu+1)(2n+1)) (nu lam n;000)(nu lam n;-m 0 m), lambda = |n-nu| .. n+nu step 2
  std::vector<double> coef_;
  std::vector<uint32_t> offset_;
  size_t slot(int m, int nu, int n) const;
};

// coefficients of the orthonormal Legendre recurrences used on the device (special.cpp:80-95):
//   diag[m]   = -sqrt((2m+1)/(2m))            Pbar_m^m   = diag[m] * sin(theta) * Pbar_{m-1}^{m-1}
//   sub[m]    =  sqrt(2m+3)                   Pbar_{m+1}^m = sub[m] * cos(theta) * Pbar_m^m
//   a[n,m], b[n,m]                            Pbar_n^m = a x Pbar_{n-1}^m - b Pbar_{n-2}^m
// a/b indexed by n*(n+1)/2 + m
void build_legendre_coefficients(int order, float* diag, float* sub, float* a, float* b);

}  // namespace hfmm_b200
