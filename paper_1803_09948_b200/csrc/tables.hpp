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
// coefficients) with one aligned 16-byte load:
//   rotation block n : (2n+1) rows of rot_row_stride(n) floats, E_n[m][m'] at row m+n, column m'+n
//   coaxial block m  : (P+1-m) rows of coax_row_stride(P,m) complex, Chat^m[n][nu] at row n-m,
//                      column nu-m
// padding entries are zero.
HFMM_HD constexpr int rot_row_stride(int n) { return (2 * n + 1 + 3) & ~3; }
HFMM_HD constexpr int rot_block_offset(int n) {
  int off = 0;
  for (int j = 0; j < n; ++j) off += (2 * j + 1) * rot_row_stride(j);
  return off;
}
HFMM_HD constexpr int rot_table_size(int p) { return rot_block_offset(p + 1); }
HFMM_HD constexpr int coax_row_stride(int p, int m) { return (p + 1 - m + 1) & ~1; }
HFMM_HD constexpr int coax_block_offset(int p, int m) {
  int off = 0;
  for (int j = 0; j < m; ++j) off += (p + 1 - j) * coax_row_stride(p, j);
  return off;
}
HFMM_HD constexpr int coax_table_size(int p) { return coax_block_offset(p, p + 1); }  // complex

// E_n[m][m'] = d^n_{m,m'}(theta), padded blocks concatenated over n; forward rotation is
//   M'_n^{m'} = sum_m E_n[m][m'] e^{i m phi} M_n^m   (then  M = R^H M' for the inverse)
void build_rotation_table(int order, double cos_theta, float* out);

enum class CoaxKind { m2l, m2m, l2l };
// Scaled coaxial coefficients Chat^m[n][nu] (complex, interleaved) for translation distance
// `dist` along +z at wavenumber k;  s_src / s_dst are the level scales of the source-side and
// destination-side expansions.
class CoaxBuilder {
 public:
  explicit CoaxBuilder(int order);
  void build(CoaxKind kind, double k, double dist, double s_src, double s_dst, float* out) const;
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
