/* oracle/hfmm_oracle.h — CPU restatement of the reference's FMM matvec path (plain C11, FP64).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER.  The product (libhfmm_b200.so) never links or loads it.
 *
 * Parity status: PINNED.  The reference ships no golden vectors; instead this
 * restatement is checked (tests/test_oracle_vs_reference.py) against the reference itself compiled
 * unmodified into oracle/_ref/libhfmm_ref.so, against fixtures that library generated
 * (tests/golden/, made by tests/golden/make_golden.py), and against the closed forms the
 * reference's own tests use (tests/test_special.cpp, tests/test_fmm.cpp).
 *
 * Scope: real wavenumber only (wave_i = 0, as in every BASELINE.json config).  Complex arrays are
 * interleaved (re, im) doubles.  Coefficient index is n*(n+1)+m (special.hpp:29).
 */
#ifndef HFMM_ORACLE_H
#define HFMM_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

/* special functions — special.cpp:16-155 */
void ho_sph_jn(int nmax, double z, double* out);            /* out[n], real */
void ho_sph_hn(int nmax, double z, double* out_re_im);      /* out[2n], out[2n+1] */
void ho_ynm(int nmax, const double dir[3], double* out_re_im);
double ho_wigner3j(int j1, int j2, int j3, int m1, int m2, int m3);

/* expansion operators — expansion.cpp:95-195 */
void ho_translation_matrix(double k, const double t[3], int order, int singular, double* out);
void ho_p2m(long n, const double* xyz, const double* q, const double center[3], double k,
            int order, double* out);
void ho_eval_expansion(int local, int order, const double* coeff, const double center[3],
                       const double point[3], double k, double out[2]);

/* tree + traversal + pipeline — octree.cpp:25-182, traversal.cpp:36-279 */
typedef struct ho_fmm ho_fmm;
ho_fmm* ho_fmm_create(long n, const double* xyz, double k, int order, int ncrit,
                      double leaf_cap, double theta, double kd_max);
void ho_fmm_destroy(ho_fmm* h);
/* same layouts as ref_fmm_counts / ref_fmm_cells / ref_fmm_body_order / ref_fmm_plan */
void ho_fmm_counts(const ho_fmm* h, long long* c);
void ho_fmm_cells(const ho_fmm* h, unsigned* out);
void ho_fmm_box(const ho_fmm* h, double* lo_w);
void ho_fmm_body_order(const ho_fmm* h, unsigned* out);
void ho_fmm_plan(const ho_fmm* h, int which, unsigned* targets, unsigned long long* offsets,
                 unsigned* sources);
/* one matvec; q/out in caller order; f32_p2p mirrors kernel::Precision::f32.  Returns 0. */
int ho_fmm_matvec(ho_fmm* h, const double* q, int f32_p2p, double* out);
void ho_fmm_seconds(const ho_fmm* h, double s[3]);
void ho_fmm_expansions(const ho_fmm* h, int which, double* out);

/* FP64 direct sum at selected targets (tests/test_fmm.cpp:59-72); target_index may be NULL */
void ho_direct_sum(long n, const double* xyz, const double* q, double k, long nt,
                   const long long* target_index, double* out);

/* restarted GMRES — gmres.cpp:35-174.  report: iterations, converged, breakdown, rhs_norm,
 * final_residual */
typedef void (*ho_matvec_cb)(void* user, long n, const double* x, double* y);
int ho_gmres(ho_matvec_cb cb, void* user, long n, const double* rhs, double rtol, int restart,
             int max_iterations, double* x, double* report, double* residuals, int residual_cap);

/* apply_operator tail — solver.cpp:340-357: y += blockdiag(patch_block) x + CSR x */
void ho_apply_corrections(long n, int ni, const double* patch_block, const unsigned* near_offset,
                          const unsigned* near_source, const double* near_delta, const double* x,
                          double* y);
/* block-Jacobi apply — solver.cpp:65-74,376-382: in-place LU solves per patch */
void ho_block_lu_solve(long npatch, int ni, const double* block_lu, const int* block_piv,
                       double* x);


/* complex wavenumber kr + i ki (common.hpp:36-40): the reference's special functions, translation
 * matrices and kernels take cplx k throughout */
ho_fmm* ho_fmm_create_complex_k(long n, const double* xyz, double kr, double ki, int order, int ncrit,
                                double leaf_cap, double theta, double kd_max);
void ho_translation_matrix_complex_k(double kr, double ki, const double t[3], int order, int singular,
                                     double* out);
/* direct sum for a complex wavenumber kr + i ki (kernel.hpp:16-23) */
void ho_direct_sum_complex_k(long n, const double* xyz, const double* q, double kr, double ki, long nt,
                             const long long* target_index, double* out);

/* ---- repartitioning loop (ref: src/partition.cpp:137-227) -------------------------------------- */
/* per-body work estimates in caller order: local = P2P partners, remote = M2L pairs of every cell above the body */
void ho_measure_weights(const ho_fmm* h, double* local, double* remote);
/* golden-section replay over [0, alpha_max]; returns 0, or 1 for invalid arguments */
int ho_update_alpha(const double* alpha, const double* runtime, int n, double alpha_max, double* next);

/* ---- correction builders (setup of the BIE operator; ref: src/solver.cpp:78-230) ---------------
 * The quadrature / interpolation tables are geometry.cpp's, passed in by the caller; field for
 * field the layout of hfmm_correction_rules in include/hfmm_cuda.h. */
typedef struct {
  int basis_count;
  int mode; /* 0 none, 1 self_only, 2 self_near */
  unsigned long long n_patches;
  const double* nodes;      /* n_patches x 6 x 3 */
  const double* sample_ref; /* ni x 2 */
  const double* far_weight; /* ni */
  double near_patch_distance;
  int near_npts;
  const double* near_pts;   /* near_npts x 3 */
  const double* near_basis; /* near_npts x ni */
  const int* self_npts;     /* ni */
  const double* self_pts;
  const double* self_basis;
} ho_correction_rules;
/* sample positions (build_system, solver.cpp:283-294): xyz[n_patches * ni][3] */
void ho_correction_samples(const ho_correction_rules* r, double* xyz);
/* returns 0, or 1 when a self block is singular; block_lu / block_piv may be null when mode == 0 */
int ho_build_patch_blocks(const ho_correction_rules* r, double kr, double ki, double* patch_block,
                          double* block_lu, int* block_piv);
/* near_offset[n + 1]; *near_source is malloc'd (release with ho_free); returns nnz */
long ho_build_near_lists(const ho_correction_rules* r, unsigned* near_offset, unsigned** near_source);
void ho_build_near_deltas(const ho_correction_rules* r, double kr, double ki, const unsigned* near_offset,
                          const unsigned* near_source, double* near_delta);
void ho_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
