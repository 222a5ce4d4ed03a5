/*
 * gliosim_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference gliosim hot path (the exponential-Euler
 * step and everything it calls), used as the CHECKER for the CUDA product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.  The product (paper_2402_02273_b200) never links,
 * imports or executes it.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function below
 * bit-for-bit against golden vectors produced by the reference itself
 * (oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile;
 * generator tests/golden/make_golden.py).
 *
 * Arithmetic model: x86-64 SSE2 doubles, no FMA contraction
 * (compile with -ffp-contract=off), evaluation order exactly as the reference.
 */
#ifndef GLIOSIM_ORACLE_H
#define GLIOSIM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_EINVAL = 1, OR_ENUMERIC = 2, OR_EDATA = 3 };

enum { OR_OP_STENCIL = 0, OR_OP_CSR = 1, OR_OP_BORDERED = 2 };

#define OR_MAX_LOGGED_STAGES 256

/* A linear operator the Taylor driver can apply.  STENCIL is the matrix-free
 * restatement of assemble_diffusion (stencil.cpp:5-43) applied in CSR column
 * order (sparse.cpp:54-58); CSR is a plain SparseOperator; BORDERED is the
 * phi1v augmented operator [[A, b/gamma],[0,0]] (expact.cpp:124-142). */
typedef struct or_op {
    int kind;
    /* STENCIL */
    int nx, ny, nz;
    double h;
    const double* d; /* per-voxel diffusion, x-fastest */
    /* CSR */
    int64_t dim;
    const int64_t* offs;
    const int32_t* cols;
    const double* vals;
    /* BORDERED */
    const struct or_op* base;
    const double* border; /* b_i / gamma, length base dim */
    const double* b;      /* original b, entry exists iff b_i != 0 */
} or_op;

/* What one expmv / phi1v / step did: (s, m), terms used per stage, the norms. */
typedef struct or_log {
    int s, m;
    int branch;          /* 0 taylor, 1 t==0, 2 bnorm==0, 3 small-norm */
    int64_t total_terms; /* Taylor terms (SpMVs inside expmv) */
    int terms[OR_MAX_LOGGED_STAGES];
    double bnorm, anorm, coln, gamma, norm_tA;
} or_log;

/* ---- material map (imaging.cpp:65-72, 118-153) ---- */
int or_classify(int intensity, int t_air, int t_white, int t_gray);
int or_nearest_source(int i, int n, int src);
void or_resample(const uint8_t* stack, int w, int hgt, int slices, int nx, int ny, int nz,
                 int t_air, int t_white, int t_gray, uint8_t* labels);
void or_diffusion_from_labels(const uint8_t* labels, int64_t n, double d_white, double d_gray,
                              double* d);

/* ---- operator ---- */
int64_t or_op_dim(const or_op* op);
void or_op_apply(const or_op* op, const double* x, double* y);
double or_op_one_norm(const or_op* op);
/* Column sums of the stencil operator (sparse.cpp:36-38 restated), length n. */
void or_stencil_colsums(const or_op* op, double* colsum);

/* ---- exponential action (expact.cpp:29-153) ---- */
int or_select_params(double norm_tA, double tol, int* s, int* m);
int or_expmv(double t, const or_op* op, const double* b, double tol, double* out, or_log* log);
/* bnorm_override / coln_override: NULL = compute as the reference does (sequential sums);
 * non-NULL = use the given value (lets the tests reproduce the GPU's tree-reduced sums
 * and then demand bitwise equality of everything downstream). */
int or_phi1v_ex(double t, const or_op* op, const double* b, double tol, double* out, or_log* log,
                const double* bnorm_override, const double* coln_override);
int or_phi1v(double t, const or_op* op, const double* b, double tol, double* out, or_log* log);

/* ---- integrator (integrator.cpp:32-89) ---- */
int or_step_ex(const or_op* a, const double* u, double rho, double tau, double tol, double* out,
               or_log* log, const double* bnorm_override, const double* coln_override);
int or_step(const or_op* a, const double* u, double rho, double tau, double tol, double* out,
            or_log* log);
void or_seed_initial(int nx, int ny, int nz, double h, const double origin[3], double amplitude,
                     double width, const double center[3], const double* d_mask, double* u);
/* out[0]=total_mass out[1]=max out[2]=min out[3]=radius */
void or_compute_metrics(const double* u, int nx, int ny, int nz, double h, const double origin[3],
                        const double center[3], double front_threshold, double out[4]);
/* n_steps steps of u in place; metrics[(n_steps+1)*4]; logs[n_steps] may be NULL. */
int or_run(const or_op* a, double* u, int n_steps, double rho, double tau, double tol,
           const double origin[3], const double center[3], double front_threshold,
           double* metrics, or_log* logs);

#ifdef __cplusplus
}
#endif

#endif
