/*
 * gliosim_oracle.c -- TEST INFRASTRUCTURE ONLY (see gliosim_oracle.h).
 *
 * CPU restatement of the reference gliosim exponential-Euler hot path in plain
 * C.  Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Evaluation order, operation by operation, follows
 * the reference so results are bit-identical to it (compiled with
 * -ffp-contract=off; the reference's x86-64 build has no FMA).
 */
#include "gliosim_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* std::max(a, b) == (a < b) ? b : a  -- NaN in b is dropped, as in the reference. */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------------ */
/* material map                                                              */
/* ------------------------------------------------------------------------ */

/* imaging.cpp:118-123 */
int or_classify(int intensity, int t_air, int t_white, int t_gray) {
    if (intensity <= t_air) return 0;   /* Air */
    if (intensity <= t_white) return 1; /* WhiteMatter */
    if (intensity <= t_gray) return 2;  /* GrayMatter */
    return 3;                           /* Skull */
}

/* imaging.cpp:65-72: nearest source index, exact halves round down. */
int or_nearest_source(int i, int n, int src) {
    if (n <= 1 || src <= 1) return 0;
    double f = (double)i * (src - 1) / (n - 1);
    int s = (int)ceil(f - 0.5);
    if (s < 0) s = 0;
    if (s > src - 1) s = src - 1;
    return s;
}

/* imaging.cpp:125-141 (stack.at: imaging.hpp:21-25) */
void or_resample(const uint8_t* stack, int w, int hgt, int slices, int nx, int ny, int nz,
                 int t_air, int t_white, int t_gray, uint8_t* labels) {
    for (int k = 0; k < nz; ++k) {
        int sz = or_nearest_source(k, nz, slices);
        for (int j = 0; j < ny; ++j) {
            int sy = or_nearest_source(j, ny, hgt);
            for (int i = 0; i < nx; ++i) {
                int sx = or_nearest_source(i, nx, w);
                size_t v = (size_t)i + (size_t)j * nx + (size_t)k * nx * ny;
                uint8_t px = stack[(size_t)sx + (size_t)sy * w + (size_t)sz * w * hgt];
                labels[v] = (uint8_t)or_classify(px, t_air, t_white, t_gray);
            }
        }
    }
}

/* imaging.cpp:143-153 */
void or_diffusion_from_labels(const uint8_t* labels, int64_t n, double d_white, double d_gray,
                              double* d) {
    for (int64_t v = 0; v < n; ++v) {
        switch (labels[v]) {
            case 1: d[v] = d_white; break;
            case 2: d[v] = d_gray; break;
            default: d[v] = 0.0; break;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* operators                                                                 */
/* ------------------------------------------------------------------------ */

int64_t or_op_dim(const or_op* op) {
    switch (op->kind) {
        case OR_OP_STENCIL: return (int64_t)op->nx * op->ny * op->nz;
        case OR_OP_CSR: return op->dim;
        default: return or_op_dim(op->base) + 1;
    }
}

/* Row v of assemble_diffusion (stencil.cpp:16-37) after CsrBuilder::push_row sorts
 * it by column (sparse.cpp:90-91): columns v-sz, v-sy, v-1, v, v+1, v+sy, v+sz,
 * off-diagonal w = d_v * (1/(h*h)), diagonal (-cnt) * w; empty when d_v == 0.
 * Accumulated as SparseOperator::apply does (sparse.cpp:54-58). */
static double stencil_row(const or_op* op, int64_t v, int i, int j, int k, const double* x) {
    const double dv = op->d[v];
    if (!(dv != 0.0)) return 0.0; /* empty row (stencil.cpp:22) */
    const double inv_h2 = 1.0 / (op->h * op->h);
    const int64_t sy = op->nx, sz = (int64_t)op->nx * op->ny;
    const double w = dv * inv_h2;
    const int hx0 = i > 0, hx1 = i < op->nx - 1;
    const int hy0 = j > 0, hy1 = j < op->ny - 1;
    const int hz0 = k > 0, hz1 = k < op->nz - 1;
    const int cnt = hx0 + hx1 + hy0 + hy1 + hz0 + hz1;
    const double diag = -cnt * w; /* stencil.cpp:36: (double)(-neighbors) * w */
    double acc = 0.0;
    if (hz0) acc += w * x[v - sz];
    if (hy0) acc += w * x[v - sy];
    if (hx0) acc += w * x[v - 1];
    acc += diag * x[v];
    if (hx1) acc += w * x[v + 1];
    if (hy1) acc += w * x[v + sy];
    if (hz1) acc += w * x[v + sz];
    return acc;
}

/* sparse.cpp:43-58 (row loop; threading does not change results, sparse.hpp:27-29) */
void or_op_apply(const or_op* op, const double* x, double* y) {
    if (op->kind == OR_OP_STENCIL) {
        int64_t v = 0;
        for (int k = 0; k < op->nz; ++k)
            for (int j = 0; j < op->ny; ++j)
                for (int i = 0; i < op->nx; ++i, ++v) y[v] = stencil_row(op, v, i, j, k, x);
    } else if (op->kind == OR_OP_CSR) {
        for (int64_t r = 0; r < op->dim; ++r) {
            double acc = 0.0;
            for (int64_t p = op->offs[r]; p < op->offs[r + 1]; ++p) acc += op->vals[p] * x[op->cols[p]];
            y[r] = acc;
        }
    } else {
        /* Bordered row i: base row entries, then (n, b_i/gamma) iff b_i != 0 -- it has
         * the largest column so it is accumulated last (expact.cpp:133-141). Row n is
         * empty (expact.cpp:141). */
        const int64_t n = or_op_dim(op->base);
        if (op->base->kind == OR_OP_STENCIL) {
            const or_op* s = op->base;
            int64_t v = 0;
            for (int k = 0; k < s->nz; ++k)
                for (int j = 0; j < s->ny; ++j)
                    for (int i = 0; i < s->nx; ++i, ++v) {
                        double acc = stencil_row(s, v, i, j, k, x);
                        if (op->b[v] != 0.0) acc += op->border[v] * x[n];
                        y[v] = acc;
                    }
        } else {
            const or_op* c = op->base;
            for (int64_t r = 0; r < n; ++r) {
                double acc = 0.0;
                for (int64_t p = c->offs[r]; p < c->offs[r + 1]; ++p) acc += c->vals[p] * x[c->cols[p]];
                if (op->b[r] != 0.0) acc += op->border[r] * x[n];
                y[r] = acc;
            }
        }
        y[n] = 0.0;
    }
}

/* Stencil column sums in CSR storage order (sparse.cpp:36-38): column c collects
 * |a_rc| from rows r = c-sz, c-sy, c-1, c, c+1, c+sy, c+sz (ascending r). */
void or_stencil_colsums(const or_op* op, double* colsum) {
    const int64_t n = (int64_t)op->nx * op->ny * op->nz;
    const double inv_h2 = 1.0 / (op->h * op->h);
    const int64_t sy = op->nx, sz = (int64_t)op->nx * op->ny;
    int64_t c = 0;
    for (int k = 0; k < op->nz; ++k)
        for (int j = 0; j < op->ny; ++j)
            for (int i = 0; i < op->nx; ++i, ++c) {
                double s = 0.0;
                /* row r = c - sz links to c via its +z neighbour (exists: k > 0) */
                if (k > 0 && op->d[c - sz] != 0.0) s += fabs(op->d[c - sz] * inv_h2);
                if (j > 0 && op->d[c - sy] != 0.0) s += fabs(op->d[c - sy] * inv_h2);
                if (i > 0 && op->d[c - 1] != 0.0) s += fabs(op->d[c - 1] * inv_h2);
                if (op->d[c] != 0.0) {
                    const int cnt = (i > 0) + (i < op->nx - 1) + (j > 0) + (j < op->ny - 1) +
                                    (k > 0) + (k < op->nz - 1);
                    const double w = op->d[c] * inv_h2;
                    s += fabs(-cnt * w);
                }
                if (i < op->nx - 1 && op->d[c + 1] != 0.0) s += fabs(op->d[c + 1] * inv_h2);
                if (j < op->ny - 1 && op->d[c + sy] != 0.0) s += fabs(op->d[c + sy] * inv_h2);
                if (k < op->nz - 1 && op->d[c + sz] != 0.0) s += fabs(op->d[c + sz] * inv_h2);
                colsum[c] = s;
            }
    (void)n;
}

/* sparse.cpp:36-40: exact 1-norm = max absolute column sum. */
double or_op_one_norm(const or_op* op) {
    double norm = 0.0;
    if (op->kind == OR_OP_STENCIL) {
        const int64_t n = or_op_dim(op);
        double* cs = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        or_stencil_colsums(op, cs);
        for (int64_t c = 0; c < n; ++c) norm = smax(norm, cs[c]);
        free(cs);
    } else if (op->kind == OR_OP_CSR) {
        double* cs = (double*)calloc((size_t)(op->dim > 0 ? op->dim : 1), sizeof(double));
        for (int64_t p = 0; p < op->offs[op->dim]; ++p) cs[op->cols[p]] += fabs(op->vals[p]);
        for (int64_t c = 0; c < op->dim; ++c) norm = smax(norm, cs[c]);
        free(cs);
    } else {
        /* Columns < n carry exactly the base column sums (the border lives in column n);
         * column n sums |b_i/gamma| over b_i != 0 in row order. */
        const int64_t n = or_op_dim(op->base);
        double coln = 0.0;
        for (int64_t i = 0; i < n; ++i)
            if (op->b[i] != 0.0) coln += fabs(op->border[i]);
        norm = smax(or_op_one_norm(op->base), coln);
    }
    return norm;
}

/* ------------------------------------------------------------------------ */
/* exponential action                                                        */
/* ------------------------------------------------------------------------ */

#define OR_MAX_TAYLOR_DEGREE 55 /* expact.hpp:39 */

/* expact.cpp:29-61 */
int or_select_params(double norm_tA, double tol, int* s_out, int* m_out) {
    if (!isfinite(norm_tA) || norm_tA < 0.0) return OR_EINVAL;
    if (!(tol > 0.0 && tol < 1.0)) return OR_EINVAL;
    *s_out = 1;
    *m_out = 1;
    if (norm_tA == 0.0) return OR_OK;
    const double r_cap = 6.0;
    double best_cost = -1.0;
    for (int m = 1; m <= OR_MAX_TAYLOR_DEGREE; ++m) {
        double r = exp((log(tol) + lgamma(m + 2.0)) / (m + 1.0));
        r = smin(r, r_cap);
        const double stages = smax(1.0, ceil(norm_tA / r));
        if (stages > 2e9) continue;
        const double cost = stages * m;
        if (best_cost < 0.0 || cost < best_cost) {
            best_cost = cost;
            *s_out = (int)stages;
            *m_out = m;
        }
    }
    if (best_cost < 0.0) return OR_ENUMERIC;
    return OR_OK;
}

/* expact.cpp:15-19 */
static double inf_norm(const double* v, int64_t n) {
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) m = smax(m, fabs(v[i]));
    return m;
}

/* expact.cpp:63-99.  op_norm: NULL = op's exact 1-norm (expact.cpp:71). */
static int expmv_impl(double t, const or_op* op, const double* b, double tol, double* out,
                      or_log* log, const double* op_norm) {
    const int64_t n = or_op_dim(op);
    if (!(tol > 0.0 && tol < 1.0)) return OR_EINVAL;
    if (log) {
        memset(log, 0, sizeof *log);
        log->s = log->m = 1;
    }
    if (t == 0.0) {
        memcpy(out, b, sizeof(double) * (size_t)n);
        if (log) log->branch = 1;
        return OR_OK;
    }
    const double norm_tA = fabs(t) * (op_norm ? *op_norm : or_op_one_norm(op));
    int s = 1, m = 1;
    int rc = or_select_params(norm_tA, tol, &s, &m);
    if (rc) return rc;
    const double tau = t / s;
    if (log) {
        log->s = s;
        log->m = m;
        log->norm_tA = norm_tA;
    }
    double* f = out;
    double* term = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* scratch = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    memcpy(f, b, sizeof(double) * (size_t)n);
    memcpy(term, b, sizeof(double) * (size_t)n);
    rc = OR_OK;
    for (int stage = 0; stage < s && rc == OR_OK; ++stage) {
        double prev = inf_norm(term, n);
        int used = 0;
        for (int j = 1; j <= m; ++j) {
            or_op_apply(op, term, scratch);
            ++used;
            const double c = tau / j;
            for (int64_t i = 0; i < n; ++i) {
                term[i] = c * scratch[i];
                f[i] += term[i];
            }
            const double cur = inf_norm(term, n);
            const double fn = inf_norm(f, n);
            if (!isfinite(cur) || !isfinite(fn)) {
                rc = OR_ENUMERIC; /* expact.cpp:90-91 */
                break;
            }
            if (prev + cur <= tol * fn) break; /* expact.cpp:93 */
            prev = cur;
        }
        if (log) {
            log->total_terms += used;
            if (stage < OR_MAX_LOGGED_STAGES) log->terms[stage] = used;
        }
        memcpy(term, f, sizeof(double) * (size_t)n);
    }
    free(term);
    free(scratch);
    return rc;
}

int or_expmv(double t, const or_op* op, const double* b, double tol, double* out, or_log* log) {
    return expmv_impl(t, op, b, tol, out, log, NULL);
}

/* expact.cpp:101-153 */
int or_phi1v_ex(double t, const or_op* op, const double* b, double tol, double* out, or_log* log,
                const double* bnorm_override, const double* coln_override) {
    const int64_t n = or_op_dim(op);
    if (!(tol > 0.0 && tol < 1.0)) return OR_EINVAL;
    if (log) {
        memset(log, 0, sizeof *log);
        log->s = log->m = 1;
    }
    if (t == 0.0) {
        memcpy(out, b, sizeof(double) * (size_t)n);
        if (log) log->branch = 1;
        return OR_OK;
    }
    double bnorm = 0.0;
    for (int64_t i = 0; i < n; ++i) bnorm += fabs(b[i]); /* expact.cpp:21-25 */
    if (bnorm_override) bnorm = *bnorm_override;
    if (log) log->bnorm = bnorm;
    if (bnorm == 0.0) {
        memset(out, 0, sizeof(double) * (size_t)n);
        if (log) log->branch = 2;
        return OR_OK;
    }
    const double anorm = or_op_one_norm(op);
    if (log) log->anorm = anorm;
    if (fabs(t) * anorm <= 1e-8) { /* expact.cpp:114-122 */
        or_op_apply(op, b, out);
        for (int64_t i = 0; i < n; ++i) out[i] = b[i] + 0.5 * t * out[i];
        if (log) log->branch = 3;
        return OR_OK;
    }
    const double gamma = bnorm / anorm;
    double* border = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) border[i] = (b[i] != 0.0) ? b[i] / gamma : 0.0;
    or_op bordered;
    memset(&bordered, 0, sizeof bordered);
    bordered.kind = OR_OP_BORDERED;
    bordered.base = op;
    bordered.border = border;
    bordered.b = b;

    double* unit = (double*)calloc((size_t)n + 1, sizeof(double));
    double* y = (double*)malloc(sizeof(double) * ((size_t)n + 1));
    unit[n] = 1.0;
    /* Bordered 1-norm: columns < n carry A's column sums, column n is coln
     * (sparse.cpp:36-40 over the bordered CSR) -- or the override. */
    double coln = 0.0;
    for (int64_t i = 0; i < n; ++i)
        if (b[i] != 0.0) coln += fabs(border[i]);
    if (coln_override) coln = *coln_override;
    const double bnorm1 = smax(anorm, coln);
    or_log tmp;
    int rc = expmv_impl(t, &bordered, unit, tol, y, &tmp, &bnorm1);
    if (log) {
        log->s = tmp.s;
        log->m = tmp.m;
        log->norm_tA = tmp.norm_tA;
        log->total_terms = tmp.total_terms;
        memcpy(log->terms, tmp.terms, sizeof tmp.terms);
        log->coln = coln;
        log->gamma = gamma;
    }
    if (rc == OR_OK) {
        const double scale = gamma / t; /* expact.cpp:150-151 */
        for (int64_t i = 0; i < n; ++i) out[i] = scale * y[i];
    }
    free(border);
    free(unit);
    free(y);
    return rc;
}

int or_phi1v(double t, const or_op* op, const double* b, double tol, double* out, or_log* log) {
    return or_phi1v_ex(t, op, b, tol, out, log, NULL, NULL);
}

/* ------------------------------------------------------------------------ */
/* integrator                                                                */
/* ------------------------------------------------------------------------ */

/* integrator.cpp:52-63 */
int or_step_ex(const or_op* a, const double* u, double rho, double tau, double tol, double* out,
               or_log* log, const double* bnorm_override, const double* coln_override) {
    const int64_t n = or_op_dim(a);
    double* g = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* incr = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    or_op_apply(a, u, g);
    for (int64_t i = 0; i < n; ++i) g[i] += rho * u[i] * (1.0 - u[i]);
    int rc = or_phi1v_ex(tau, a, g, tol, incr, log, bnorm_override, coln_override);
    if (rc == OR_OK)
        for (int64_t i = 0; i < n; ++i) out[i] = u[i] + tau * incr[i];
    free(g);
    free(incr);
    return rc;
}

int or_step(const or_op* a, const double* u, double rho, double tau, double tol, double* out,
            or_log* log) {
    return or_step_ex(a, u, rho, tau, tol, out, log, NULL, NULL);
}

/* integrator.cpp:23-29 (sq_dist) */
static inline double sq_dist(const double p[3], const double q[3]) {
    const double dx = p[0] - q[0];
    const double dy = p[1] - q[1];
    const double dz = p[2] - q[2];
    return dx * dx + dy * dy + dz * dz;
}

/* integrator.cpp:32-50; Grid::point grid.hpp:21-23 */
void or_seed_initial(int nx, int ny, int nz, double h, const double origin[3], double amplitude,
                     double width, const double center[3], const double* d_mask, double* u) {
    int64_t v = 0;
    for (int k = 1; k <= nz; ++k)
        for (int j = 1; j <= ny; ++j)
            for (int i = 1; i <= nx; ++i, ++v) {
                const double p[3] = {origin[0] + (i - 1) * h, origin[1] + (j - 1) * h,
                                     origin[2] + (k - 1) * h};
                u[v] = amplitude * exp(-width * sq_dist(p, center));
                if (d_mask && d_mask[v] == 0.0) u[v] = 0.0;
            }
}

/* integrator.cpp:65-89 */
void or_compute_metrics(const double* u, int nx, int ny, int nz, double h, const double origin[3],
                        const double center[3], double front_threshold, double out[4]) {
    const int64_t n = (int64_t)nx * ny * nz;
    double sum = 0.0;
    double max_u = n == 0 ? 0.0 : u[0];
    double min_u = max_u;
    double r2 = 0.0;
    int64_t v = 0;
    for (int k = 1; k <= nz; ++k)
        for (int j = 1; j <= ny; ++j)
            for (int i = 1; i <= nx; ++i, ++v) {
                sum += u[v];
                max_u = smax(max_u, u[v]);
                min_u = smin(min_u, u[v]);
                if (u[v] >= front_threshold) {
                    const double p[3] = {origin[0] + (i - 1) * h, origin[1] + (j - 1) * h,
                                         origin[2] + (k - 1) * h};
                    r2 = smax(r2, sq_dist(p, center));
                }
            }
    const double cell = h * h * h;
    out[0] = cell * sum;
    out[1] = max_u;
    out[2] = min_u;
    out[3] = sqrt(r2);
}

/* integrator.cpp:91-138 (no hooks; snapshots are the caller's business) */
int or_run(const or_op* a, double* u, int n_steps, double rho, double tau, double tol,
           const double origin[3], const double center[3], double front_threshold,
           double* metrics, or_log* logs) {
    const int64_t n = or_op_dim(a);
    double* next = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (metrics)
        or_compute_metrics(u, a->nx, a->ny, a->nz, a->h, origin, center, front_threshold, metrics);
    int rc = OR_OK;
    for (int s = 1; s <= n_steps; ++s) {
        rc = or_step(a, u, rho, tau, tol, next, logs ? &logs[s - 1] : NULL);
        if (rc) break;
        memcpy(u, next, sizeof(double) * (size_t)n);
        if (metrics)
            or_compute_metrics(u, a->nx, a->ny, a->nz, a->h, origin, center, front_threshold,
                               metrics + 4 * s);
    }
    free(next);
    return rc;
}
