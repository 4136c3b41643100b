/*
 * sk_oracle.c -- CPU ORACLE (test infrastructure only; see sk_oracle.h).
 *
 * Plain-C restatement of the reference sLdG step. Every function names the
 * reference file:line it restates; expressions keep the reference's
 * left-to-right evaluation order so results are bitwise comparable. Build with
 * -ffp-contract=off (oracle/Makefile) -- the reference is compiled without
 * -march, hence without FMA.
 */
#include "sk_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static char g_err[512];
static long g_err_step = 0;
const char* sko_last_error(void) { return g_err; }
long sko_last_error_step(void) { return g_err_step; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* std::max / std::min semantics (first argument wins ties) */
static inline double dmax2(double a, double b) { return (a < b) ? b : a; }
static inline double dmin2(double a, double b) { return (b < a) ? b : a; }
static inline int imax2(int a, int b) { return (a < b) ? b : a; }
static inline int imin2(int a, int b) { return (b < a) ? b : a; }

/* ======================================================================
 * basis  (core/src/basis.cpp)
 * ==================================================================== */

/* basis.cpp:14-25 legendre_with_derivative */
static void legendre_wd(int n, double t, double* P, double* dP) {
    double p0 = 1.0, p1 = t;
    if (n == 0) {
        *P = 1.0;
        *dP = 0.0;
        return;
    }
    for (int j = 2; j <= n; ++j) {
        double p2 = ((double)(2 * j - 1) * t * p1 - (double)(j - 1) * p0) / (double)j;
        p0 = p1;
        p1 = p2;
    }
    *P = p1;
    *dP = (double)n * (t * p1 - p0) / (t * t - 1.0);
}

/* basis.cpp:29-48 gauss_legendre */
int sko_gauss_legendre(int k, double* nodes, double* weights) {
    if (k < 0) return fail(SKO_ERR_RUNTIME, "gauss_legendre: degree must be >= 0");
    const int n = k + 1;
    for (int i = 0; i < n; ++i) {
        double t = -cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int iter = 0; iter < 100; ++iter) {
            double P, dP;
            legendre_wd(n, t, &P, &dP);
            double dt = P / dP;
            t -= dt;
            if (fabs(dt) < 1e-15) break;
        }
        double P, dP;
        legendre_wd(n, t, &P, &dP);
        nodes[i] = 0.5 * (t + 1.0);
        weights[i] = 1.0 / ((1.0 - t * t) * dP * dP);
    }
    return SKO_OK;
}

/* basis.cpp:50-91 ReferenceBasis ctor */
int sko_basis_init(sko_basis* b, int k) {
    if (k < 0 || k > SKO_MAXP - 1) return fail(SKO_ERR_RUNTIME, "basis: degree out of range");
    memset(b, 0, sizeof *b);
    b->k = k;
    b->p = k + 1;
    int rc = sko_gauss_legendre(k, b->nodes, b->weights);
    if (rc) return rc;
    const int p = b->p;
    for (int i = 0; i < p; ++i) {
        b->bary[i] = 1.0;
        for (int j = 0; j < p; ++j)
            if (j != i) b->bary[i] /= (b->nodes[i] - b->nodes[j]);
    }
    for (int m = 0; m < p; ++m) {
        double row_sum = 0.0;
        for (int n2 = 0; n2 < p; ++n2) {
            if (n2 == m) continue;
            double d = b->bary[n2] / b->bary[m] / (b->nodes[m] - b->nodes[n2]);
            b->diff[m * p + n2] = d;
            row_sum += d;
        }
        b->diff[m * p + m] = -row_sum;
    }
    for (int n2 = 0; n2 < p; ++n2) {
        double c[SKO_MAXP + 1];
        for (int d = 0; d < p; ++d) c[d] = 0.0;
        c[0] = b->bary[n2];
        int deg = 0;
        for (int j = 0; j < p; ++j) {
            if (j == n2) continue;
            for (int d = deg; d >= 0; --d) {
                c[d + 1] += c[d];
                c[d] *= -b->nodes[j];
            }
            ++deg;
        }
        for (int d = 0; d < p; ++d) b->mono[d * p + n2] = c[d];
    }
    return SKO_OK;
}

/* basis.cpp:102-108 */
double sko_lagrange(const sko_basis* b, int n, double xi) {
    double v = b->bary[n];
    for (int j = 0; j < b->p; ++j)
        if (j != n) v *= (xi - b->nodes[j]);
    return v;
}

/* basis.cpp:110-121 */
double sko_lagrange_derivative(const sko_basis* b, int n, double xi) {
    double acc = 0.0;
    for (int j = 0; j < b->p; ++j) {
        if (j == n) continue;
        double term = 1.0;
        for (int i = 0; i < b->p; ++i)
            if (i != n && i != j) term *= (xi - b->nodes[i]);
        acc += term;
    }
    return b->bary[n] * acc;
}

/* basis.cpp:123-134 second barycentric form */
double sko_evaluate(const sko_basis* b, const double* u, double xi) {
    double num = 0.0, den = 0.0;
    for (int n = 0; n < b->p; ++n) {
        if (xi == b->nodes[n]) return u[n];
        double t = b->bary[n] / (xi - b->nodes[n]);
        num += t * u[n];
        den += t;
    }
    return num / den;
}

/* basis.cpp:136-140 */
double sko_mean(const sko_basis* b, const double* u) {
    double acc = 0.0;
    for (int j = 0; j < b->p; ++j) acc += b->weights[j] * u[j];
    return acc;
}

/* basis.cpp:142-150 */
double sko_integrate(const sko_basis* b, const double* u, double a, double bb) {
    double acc = 0.0;
    const double len = bb - a;
    for (int q = 0; q < b->p; ++q) {
        double xi = a + len * b->nodes[q];
        acc += b->weights[q] * sko_evaluate(b, u, xi);
    }
    return acc * len;
}

/* basis.cpp:152-161 */
void sko_interval_moments(const sko_basis* b, double a, double bb, double* m) {
    const double len = bb - a;
    for (int n = 0; n < b->p; ++n) m[n] = 0.0;
    for (int q = 0; q < b->p; ++q) {
        double xi = a + len * b->nodes[q];
        for (int n = 0; n < b->p; ++n) m[n] += b->weights[q] * len * sko_lagrange(b, n, xi);
    }
}

/* basis.cpp:163-170 */
void sko_to_monomial(const sko_basis* b, const double* u, double* c) {
    const int p = b->p;
    for (int d = 0; d < p; ++d) {
        double acc = 0.0;
        for (int n = 0; n < p; ++n) acc += b->mono[d * p + n] * u[n];
        c[d] = acc;
    }
}

/* basis.cpp:172-215 extremum_on; sign=+1 max, -1 min */
static int better(double x, double y, int sign) { return sign > 0 ? (x > y) : (x < y); }

static double extremum_on(const sko_basis* b, const double* u, double a, double bb, int sign) {
    double best = sko_evaluate(b, u, a);
    if (bb == a) return best;
    double vb = sko_evaluate(b, u, bb);
    if (better(vb, best, sign)) best = vb;
    const int k = b->k;
    if (k <= 1) return best;
    if (k <= 3) {
        double c[4] = {0, 0, 0, 0};
        sko_to_monomial(b, u, c);
        double qa = 3.0 * c[3], qb = 2.0 * c[2], qc = c[1];
        double cand[2];
        int nc = 0;
        if (fabs(qa) > 0.0) {
            double disc = qb * qb - 4.0 * qa * qc;
            if (disc >= 0.0) {
                double r = sqrt(disc);
                cand[nc++] = (-qb + r) / (2.0 * qa);
                cand[nc++] = (-qb - r) / (2.0 * qa);
            }
        } else if (fabs(qb) > 0.0) {
            cand[nc++] = -qc / qb;
        }
        for (int i = 0; i < nc; ++i) {
            double x = cand[i];
            if (x > a && x < bb) {
                double v = sko_evaluate(b, u, x);
                if (better(v, best, sign)) best = v;
            }
        }
        return best;
    }
    for (int j = 0; j < 33; ++j) {
        double t = cos(M_PI * (2 * j + 1) / 66.0);
        double x = 0.5 * (a + bb) + 0.5 * (bb - a) * t;
        double v = sko_evaluate(b, u, x);
        if (better(v, best, sign)) best = v;
    }
    return best;
}

double sko_max_on(const sko_basis* b, const double* u, double a, double bb) {
    return extremum_on(b, u, a, bb, +1);
}
double sko_min_on(const sko_basis* b, const double* u, double a, double bb) {
    return extremum_on(b, u, a, bb, -1);
}

/* ======================================================================
 * shift decomposition and matrices  (core/src/advection.cpp:14-66)
 * ==================================================================== */

void sko_decompose_shift(double speed, double dt, double dx, int* istar, double* alpha) {
    double s = -speed * dt / dx;
    double fl = floor(s);
    double al = s - fl;
    int is = (int)fl;
    if (al >= 1.0) {
        al -= 1.0;
        is += 1;
    }
    *istar = is;
    *alpha = al;
}

int sko_shift_matrices(const sko_basis* b, double alpha, double* A, double* B) {
    if (!(alpha >= 0.0 && alpha < 1.0))
        return fail(SKO_ERR_RUNTIME, "build_shift_matrices: alpha must be in [0,1)");
    const int p = b->p;
    for (int i = 0; i < p * p; ++i) A[i] = B[i] = 0.0;
    const double* xq = b->nodes;
    const double* wq = b->weights;
    double len_a = 1.0 - alpha;
    for (int q = 0; q < p; ++q) {
        double xi = len_a * xq[q];
        for (int m = 0; m < p; ++m) {
            double lm = sko_lagrange(b, m, xi);
            for (int n = 0; n < p; ++n)
                A[m * p + n] += wq[q] * len_a * sko_lagrange(b, n, xi + alpha) * lm;
        }
    }
    for (int q = 0; q < p; ++q) {
        double xi = 1.0 - alpha + alpha * xq[q];
        for (int m = 0; m < p; ++m) {
            double lm = sko_lagrange(b, m, xi);
            for (int n = 0; n < p; ++n)
                B[m * p + n] += wq[q] * alpha * sko_lagrange(b, n, alpha * xq[q]) * lm;
        }
    }
    for (int m = 0; m < p; ++m) {
        double inv_w = 1.0 / wq[m];
        for (int n = 0; n < p; ++n) {
            A[m * p + n] *= inv_w;
            B[m * p + n] *= inv_w;
        }
    }
    return SKO_OK;
}

/* ======================================================================
 * limiters  (core/src/limiters.cpp)
 * ==================================================================== */

/* limiters.cpp:14-37 LimiterConfig::parse; defaults limiters.hpp:19-27 */
int sko_limiter_parse(const char* mode, sko_limiter* c) {
    memset(c, 0, sizeof *c);
    c->threshold = 0.5;
    c->gamma_simple[0] = 0.001;
    c->gamma_simple[1] = 0.998;
    c->gamma_simple[2] = 0.001;
    c->gamma_line[0] = 0.45;
    c->gamma_line[1] = 0.1;
    c->gamma_line[2] = 0.45;
    c->epsilon = 1e-6;
    if (strcmp(mode, "none") == 0) return SKO_OK;
    if (strcmp(mode, "sldg") == 0) {
        c->inline_sldg = 1;
        return SKO_OK;
    }
    const char* plus = strchr(mode, '+');
    if (!plus) return fail(SKO_ERR_RUNTIME, "unknown limiter mode: %s", mode);
    size_t il = (size_t)(plus - mode);
    if (il == 6 && strncmp(mode, "minmod", 6) == 0)
        c->indicator = SKO_IND_MINMOD;
    else if (il == 7 && strncmp(mode, "meanerr", 7) == 0)
        c->indicator = SKO_IND_MEANERR;
    else
        return fail(SKO_ERR_RUNTIME, "unknown limiter indicator: %.*s", (int)il, mode);
    if (strcmp(plus + 1, "simple") == 0)
        c->modifier = SKO_MOD_SIMPLE;
    else if (strcmp(plus + 1, "line") == 0)
        c->modifier = SKO_MOD_LINE;
    else
        return fail(SKO_ERR_RUNTIME, "unknown limiter modifier: %s", plus + 1);
    return SKO_OK;
}

/* limiters.cpp:167-173 InlineLimiter ctor */
void sko_inline_init(sko_inline* L, const sko_basis* b, double alpha, double threshold) {
    L->alpha = alpha;
    L->threshold = threshold;
    sko_interval_moments(b, -alpha, 1.0 - alpha, L->ext_l);
    sko_interval_moments(b, 1.0 - alpha, 2.0 - alpha, L->ext_r);
}

/* limiters.cpp:175-189 */
int sko_inline_indicator(const sko_inline* L, const sko_basis* b, const double* ul,
                         const double* ur, const double* up) {
    double mean_l = sko_mean(b, ul);
    double mean_r = sko_mean(b, ur);
    double denom = dmax2(fabs(mean_l), fabs(mean_r));
    if (denom <= 0.0) return 0;
    double ext_l = 0.0, ext_r = 0.0;
    for (int n = 0; n < b->p; ++n) {
        ext_l += L->ext_l[n] * up[n];
        ext_r += L->ext_r[n] * up[n];
    }
    double ind = (fabs(ext_l - mean_l) + fabs(ext_r - mean_r)) / denom;
    return ind > L->threshold;
}

/* limiters.cpp:191-215 */
int sko_inline_clamp(const sko_inline* L, const sko_basis* b, const double* ul, const double* ur,
                     double* up) {
    int flags = 1; /* troubled */
    const double alpha = L->alpha;
    double mean_p = sko_mean(b, up);
    double wmax = dmax2(sko_max_on(b, ul, alpha, 1.0), sko_max_on(b, ur, 0.0, alpha));
    double wmin = dmin2(sko_min_on(b, ul, alpha, 1.0), sko_min_on(b, ur, 0.0, alpha));
    double pmax = sko_max_on(b, up, 0.0, 1.0);
    double pmin = sko_min_on(b, up, 0.0, 1.0);
    if ((mean_p > wmax) || (mean_p < wmin)) flags |= 4;
    double theta = 1.0;
    double dmx = pmax - mean_p;
    if (dmx != 0.0) theta = dmin2(theta, fabs((wmax - mean_p) / dmx));
    double dmn = pmin - mean_p;
    if (dmn != 0.0) theta = dmin2(theta, fabs((wmin - mean_p) / dmn));
    if (theta < 1.0) {
        for (int j = 0; j < b->p; ++j) up[j] = theta * (up[j] - mean_p) + mean_p;
        flags |= 2;
    }
    return flags;
}

/* limiters.cpp:217-222 */
int sko_inline_apply(const sko_inline* L, const sko_basis* b, const double* ul, const double* ur,
                     double* up) {
    if (!sko_inline_indicator(L, b, ul, ur, up)) return 0;
    return sko_inline_clamp(L, b, ul, ur, up);
}

/* limiters.cpp:47-51 */
double sko_minmod(double a, double b, double c) {
    if (a > 0 && b > 0 && c > 0) return dmin2(a, dmin2(b, c));
    if (a < 0 && b < 0 && c < 0) return -dmin2(-a, dmin2(-b, -c));
    return 0.0;
}

/* limiters.cpp:53-70 */
int sko_indicator_minmod(const sko_basis* b, const double* um, const double* u0, const double* up) {
    double mean_m = sko_mean(b, um);
    double mean_0 = sko_mean(b, u0);
    double mean_p = sko_mean(b, up);
    double u0_plus = sko_evaluate(b, u0, 1.0) - mean_0;
    double u0_minus = mean_0 - sko_evaluate(b, u0, 0.0);
    double d_plus = mean_p - mean_0;
    double d_minus = mean_0 - mean_m;
    double vals[7] = {fabs(mean_m), fabs(mean_0), fabs(mean_p), fabs(u0_plus),
                      fabs(u0_minus), fabs(d_plus), fabs(d_minus)};
    double scale = vals[0];
    for (int i = 1; i < 7; ++i)
        if (scale < vals[i]) scale = vals[i];
    double guard = 1e-13 * scale;
    return fabs(sko_minmod(u0_plus, d_plus, d_minus) - u0_plus) > guard ||
           fabs(sko_minmod(u0_minus, d_plus, d_minus) - u0_minus) > guard;
}

/* limiters.cpp:72-83 */
int sko_indicator_meanerr(const sko_basis* b, const double* um, const double* u0, const double* up,
                          double threshold) {
    double mean_m = sko_mean(b, um);
    double mean_0 = sko_mean(b, u0);
    double mean_p = sko_mean(b, up);
    double denom = dmax2(fabs(mean_m), dmax2(fabs(mean_0), fabs(mean_p)));
    if (denom <= 0.0) return 0;
    double ext_m = sko_integrate(b, um, 1.0, 2.0);
    double ext_p = sko_integrate(b, up, -1.0, 0.0);
    double ind = (fabs(ext_m - mean_0) + fabs(ext_p - mean_0)) / denom;
    return ind > threshold;
}

/* limiters.cpp:85-100 */
double sko_smoothness_beta(const sko_basis* b, const double* u) {
    const int p = b->p;
    double cur[SKO_MAXP], next[SKO_MAXP];
    for (int i = 0; i < p; ++i) cur[i] = u[i];
    double total = 0.0;
    for (int s = 1; s <= b->k; ++s) {
        for (int m = 0; m < p; ++m) {
            double acc = 0.0;
            for (int n = 0; n < p; ++n) acc += b->diff[m * p + n] * cur[n];
            next[m] = acc;
        }
        for (int q = 0; q < p; ++q) total += b->weights[q] * next[q] * next[q];
        for (int i = 0; i < p; ++i) cur[i] = next[i];
    }
    return total;
}

/* limiters.cpp:102-127 */
void sko_modify_simple_weno(const sko_basis* b, const double* um, const double* u0,
                            const double* up, const sko_limiter* cfg, double* out) {
    double beta_m = sko_smoothness_beta(b, um);
    double beta_0 = sko_smoothness_beta(b, u0);
    double beta_p = sko_smoothness_beta(b, up);
    double eps = cfg->epsilon;
    double wm = cfg->gamma_simple[0] / ((eps + beta_m) * (eps + beta_m));
    double w0 = cfg->gamma_simple[1] / ((eps + beta_0) * (eps + beta_0));
    double wp = cfg->gamma_simple[2] / ((eps + beta_p) * (eps + beta_p));
    double sum = wm + w0 + wp;
    wm /= sum;
    w0 /= sum;
    wp /= sum;
    double mean_0 = sko_mean(b, u0);
    double ext_mean_m = sko_integrate(b, um, 1.0, 2.0);
    double ext_mean_p = sko_integrate(b, up, -1.0, 0.0);
    for (int m = 0; m < b->p; ++m) {
        double xi = b->nodes[m];
        double cand_m = sko_evaluate(b, um, 1.0 + xi) - ext_mean_m + mean_0;
        double cand_p = sko_evaluate(b, up, xi - 1.0) - ext_mean_p + mean_0;
        out[m] = wm * cand_m + w0 * u0[m] + wp * cand_p;
    }
}

/* limiters.cpp:129-165 */
void sko_modify_line_weno(const sko_basis* b, const double* um, const double* u0, const double* up,
                          const sko_limiter* cfg, double* out) {
    const int p = b->p;
    double mean_m = sko_mean(b, um);
    double mean_0 = sko_mean(b, u0);
    double mean_p = sko_mean(b, up);
    double bm = mean_0 - mean_m, am = mean_0 - 0.5 * bm;
    double bp = mean_p - mean_0, ap = mean_0 - 0.5 * bp;
    double gm = cfg->gamma_line[0], g0 = cfg->gamma_line[1], gp = cfg->gamma_line[2];
    double pm[SKO_MAXP], pp[SKO_MAXP], p0[SKO_MAXP];
    for (int m = 0; m < p; ++m) {
        double xi = b->nodes[m];
        pm[m] = am + bm * xi;
        pp[m] = ap + bp * xi;
        p0[m] = (u0[m] - gm * pm[m] - gp * pp[m]) / g0;
    }
    double beta_m = sko_smoothness_beta(b, um);
    double beta_0 = sko_smoothness_beta(b, u0);
    double beta_p = sko_smoothness_beta(b, up);
    double tau = 0.5 * (fabs(beta_0 - beta_m) + fabs(beta_0 - beta_p));
    tau *= tau;
    double eps = cfg->epsilon;
    double wm = gm * (1.0 + tau / (eps + beta_m));
    double w0 = g0 * (1.0 + tau / (eps + beta_0));
    double wp = gp * (1.0 + tau / (eps + beta_p));
    double sum = wm + w0 + wp;
    wm /= sum;
    w0 /= sum;
    wp /= sum;
    for (int m = 0; m < p; ++m) out[m] = wm * pm[m] + w0 * p0[m] + wp * pp[m];
}

/* ======================================================================
 * grid  (core/src/grid.cpp)
 * ==================================================================== */

/* grid.cpp:9-29 */
int sko_grid_init(sko_grid* g, int nblocks, const double* left, const int* cells, const double* dx) {
    if (nblocks < 1) return fail(SKO_ERR_RUNTIME, "Grid1D: needs at least one block");
    if (nblocks > SKO_MAXB) return fail(SKO_ERR_RUNTIME, "Grid1D: too many blocks");
    memset(g, 0, sizeof *g);
    g->nblocks = nblocks;
    g->start[0] = 0;
    for (int b = 0; b < nblocks; ++b) {
        if (!(cells[b] >= 1 && dx[b] > 0))
            return fail(SKO_ERR_RUNTIME, "Grid1D: block must have cells >= 1, dx > 0");
        if (b > 0) {
            double prev_right = left[b - 1] + cells[b - 1] * dx[b - 1];
            if (!(fabs(prev_right - left[b]) <= 1e-12 * (fabs(left[b]) + dx[b - 1])))
                return fail(SKO_ERR_RUNTIME, "Grid1D: blocks must be contiguous");
            double coarse = dmax2(dx[b - 1], dx[b]);
            double fine = dmin2(dx[b - 1], dx[b]);
            double ratio = coarse / fine;
            if (!(fabs(ratio - round(ratio)) < 1e-10 && round(ratio) >= 1))
                return fail(SKO_ERR_RUNTIME,
                            "Grid1D: adjacent block widths must satisfy dx_coarse = m * dx_fine");
        }
        g->left[b] = left[b];
        g->cells[b] = cells[b];
        g->dx[b] = dx[b];
        g->ncells += cells[b];
        g->start[b + 1] = g->ncells;
    }
    return SKO_OK;
}

/* grid.cpp:31-34 */
int sko_grid_uniform(sko_grid* g, double left, double right, int cells) {
    if (!(right > left && cells >= 1))
        return fail(SKO_ERR_RUNTIME, "Grid1D::uniform: invalid extent or cell count");
    double dx = (right - left) / cells;
    return sko_grid_init(g, 1, &left, &cells, &dx);
}

/* grid.cpp:36-46 */
int sko_grid_three_block(sko_grid* g, double left, double right, int nf, int nc, int m) {
    if (!(right > left)) return fail(SKO_ERR_RUNTIME, "Grid1D::three_block: invalid extent");
    if (!(nf >= 1 && nc >= 1 && m >= 1))
        return fail(SKO_ERR_RUNTIME, "Grid1D::three_block: invalid sizes");
    double dxf = (right - left) / (2.0 * nf + (double)m * nc);
    double dxc = m * dxf;
    double lefts[3], dxs[3];
    int cells[3] = {nf, nc, nf};
    lefts[0] = left;
    dxs[0] = dxf;
    lefts[1] = left + nf * dxf;
    dxs[1] = dxc;
    lefts[2] = lefts[1] + nc * dxc;
    dxs[2] = dxf;
    return sko_grid_init(g, 3, lefts, cells, dxs);
}

/* grid.cpp:48-51 */
double sko_grid_right(const sko_grid* g) {
    int b = g->nblocks - 1;
    return g->left[b] + g->cells[b] * g->dx[b];
}

/* grid.cpp:53-57 */
int sko_grid_block_of(const sko_grid* g, int cell) {
    for (int b = 0; b < g->nblocks; ++b)
        if (cell < g->start[b + 1]) return b;
    return g->nblocks - 1;
}

/* grid.cpp:59-62 */
double sko_grid_cell_left(const sko_grid* g, int cell) {
    int b = sko_grid_block_of(g, cell);
    return g->left[b] + (cell - g->start[b]) * g->dx[b];
}

double sko_grid_cell_width(const sko_grid* g, int cell) {
    return g->dx[sko_grid_block_of(g, cell)];
}

/* ======================================================================
 * field  (core/src/field.cpp)
 * ==================================================================== */

static inline size_t fidx(const sko_field* f, int xc, int xn, int vc, int vn) {
    const int p = f->k + 1;
    return (((size_t)vc * p + vn) * f->x.ncells + xc) * p + xn;
}

static const sko_basis* basis_of(int k) {
    static sko_basis cache[SKO_MAXP + 1];
    static int init[SKO_MAXP + 1];
    if (!init[k]) {
        sko_basis_init(&cache[k], k);
        init[k] = 1;
    }
    return &cache[k];
}

/* field.cpp:32-40 */
double sko_x_node(const sko_field* f, int xc, int xn) {
    const sko_basis* b = basis_of(f->k);
    return sko_grid_cell_left(&f->x, xc) + sko_grid_cell_width(&f->x, xc) * b->nodes[xn];
}
double sko_v_node(const sko_field* f, int vc, int vn) {
    const sko_basis* b = basis_of(f->k);
    return sko_grid_cell_left(&f->v, vc) + sko_grid_cell_width(&f->v, vc) * b->nodes[vn];
}

/* field.cpp:52-68 */
double sko_mass(const sko_field* f) {
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    double acc = 0.0;
    for (int vc = 0; vc < f->v.ncells; ++vc) {
        double dv = sko_grid_cell_width(&f->v, vc);
        for (int vn = 0; vn < p; ++vn) {
            double wv = b->weights[vn] * dv;
            for (int xc = 0; xc < f->x.ncells; ++xc) {
                double dx = sko_grid_cell_width(&f->x, xc);
                for (int xn = 0; xn < p; ++xn)
                    acc += wv * b->weights[xn] * dx * f->data[fidx(f, xc, xn, vc, vn)];
            }
        }
    }
    return acc;
}

/* field.cpp:70-88 */
double sko_l2_norm(const sko_field* f) {
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    double acc = 0.0;
    for (int vc = 0; vc < f->v.ncells; ++vc) {
        double dv = sko_grid_cell_width(&f->v, vc);
        for (int vn = 0; vn < p; ++vn) {
            double wv = b->weights[vn] * dv;
            for (int xc = 0; xc < f->x.ncells; ++xc) {
                double dx = sko_grid_cell_width(&f->x, xc);
                for (int xn = 0; xn < p; ++xn) {
                    double v = f->data[fidx(f, xc, xn, vc, vn)];
                    acc += wv * b->weights[xn] * dx * v * v;
                }
            }
        }
    }
    return sqrt(acc);
}

/* Harness additions: mass()'s loop with v and v^2/2 weights. */
static double v_moment(const sko_field* f, int order) {
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    double acc = 0.0;
    for (int vc = 0; vc < f->v.ncells; ++vc) {
        double dv = sko_grid_cell_width(&f->v, vc);
        for (int vn = 0; vn < p; ++vn) {
            double wv = b->weights[vn] * dv;
            double v = sko_v_node(f, vc, vn);
            double g = order == 1 ? v : 0.5 * v * v;
            for (int xc = 0; xc < f->x.ncells; ++xc) {
                double dx = sko_grid_cell_width(&f->x, xc);
                for (int xn = 0; xn < p; ++xn)
                    acc += wv * b->weights[xn] * dx * (g * f->data[fidx(f, xc, xn, vc, vn)]);
            }
        }
    }
    return acc;
}
double sko_momentum(const sko_field* f) { return v_moment(f, 1); }
double sko_kinetic_energy(const sko_field* f) { return v_moment(f, 2); }

/* field.cpp:90-94 */
int sko_all_finite(const sko_field* f) {
    const size_t n = (size_t)f->x.ncells * f->v.ncells * (f->k + 1) * (f->k + 1);
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(f->data[i])) return 0;
    return 1;
}

/* ======================================================================
 * sweeps  (core/src/advection.cpp:68-238)
 * ==================================================================== */

static const double kZero[SKO_MAXP + 1] = {0};

/* advection.cpp:68-114 */
int sko_advect_line(const sko_basis* b, const double* A, const double* B, int istar, int bc,
                    const double* in, int gl, int n, int gr, double* out, const sko_inline* lim,
                    sko_stats* stats) {
    if (n < 1) return fail(SKO_ERR_RUNTIME, "advect_line: line must have at least one cell");
    const int p = b->p;
    const int total = gl + n + gr;
    if (bc == SKO_BC_PERIODIC && !(gl == 0 && gr == 0))
        return fail(SKO_ERR_RUNTIME, "advect_line: periodic rule needs a ghost-free line");
    for (int i = 0; i < n; ++i) {
        const double *ul, *ur;
        if (bc == SKO_BC_PERIODIC) {
            int a = ((i + istar) % n + n) % n;
            ul = in + (size_t)a * p;
            ur = in + (size_t)((a + 1) % n) * p;
        } else {
            int s = gl + i + istar;
            ul = (s >= 0 && s < total) ? in + (size_t)s * p : kZero;
            ur = (s + 1 >= 0 && s + 1 < total) ? in + (size_t)(s + 1) * p : kZero;
        }
        double* o = out + (size_t)i * p;
        for (int m = 0; m < p; ++m) {
            double acc = 0.0;
            const double* Am = A + m * p;
            const double* Bm = B + m * p;
            for (int j = 0; j < p; ++j) acc += Am[j] * ul[j] + Bm[j] * ur[j];
            o[m] = acc;
        }
        if (lim) {
            int fl = sko_inline_apply(lim, b, ul, ur, o);
            if (stats) {
                stats->inline_troubled += (fl & 1) != 0;
                stats->inline_clamped += (fl & 2) != 0;
                stats->inline_mean_outside += (fl & 4) != 0;
            }
        }
    }
    if (stats) stats->outputs += n;
    return SKO_OK;
}

typedef struct {
    int istar;
    double alpha;
    double A[SKO_MAXP * SKO_MAXP], B[SKO_MAXP * SKO_MAXP];
    sko_inline lim;
    int has_lim;
} line_plan;

/* advection.cpp:132-140 make_plan */
static void make_plan(const sko_basis* b, double speed, double tau, double dx,
                      const sko_limiter* lim, line_plan* P) {
    sko_decompose_shift(speed, tau, dx, &P->istar, &P->alpha);
    sko_shift_matrices(b, P->alpha, P->A, P->B);
    P->has_lim = lim && lim->inline_sldg;
    if (P->has_lim) sko_inline_init(&P->lim, b, P->alpha, lim->threshold);
}

/* adaptivity.cpp:132-147 */
void sko_fine_to_coarse(const sko_basis* b, const double* fine, int m, double* coarse) {
    const int p = b->p;
    for (int mm = 0; mm < p; ++mm) {
        double acc = 0.0;
        for (int j = 0; j < m; ++j) {
            const double* cell = fine + (size_t)j * p;
            for (int q = 0; q < p; ++q) {
                double xi_c = (j + b->nodes[q]) / m;
                acc += b->weights[q] / m * cell[q] * sko_lagrange(b, mm, xi_c);
            }
        }
        coarse[mm] = acc / b->weights[mm];
    }
}

/* adaptivity.cpp:149-156 */
void sko_coarse_to_fine(const sko_basis* b, const double* coarse, int m, double* fine) {
    const int p = b->p;
    for (int j = 0; j < m; ++j)
        for (int q = 0; q < p; ++q)
            fine[(size_t)j * p + q] = sko_evaluate(b, coarse, (j + b->nodes[q]) / m);
}

/* adaptivity.cpp:158-161 */
int sko_required_ghost_width(double vmax, double dt, double sqrt_mu_min, double dx_local) {
    return (int)ceil(vmax * dt / (sqrt_mu_min * dx_local)) + 1;
}

/* adaptivity.cpp:169-207 fill_ghost */
static int fill_ghost(const sko_basis* b, const sko_grid* g, int block, int left_side, int j,
                      const double* line, double* ghost) {
    const int p = b->p;
    int nbi = left_side ? block - 1 : block + 1;
    int nb_begin = g->start[nbi];
    int nb_end = nb_begin + g->cells[nbi];
    int iface = left_side ? g->start[block] : g->start[block] + g->cells[block];
    const double nb_dx = g->dx[nbi], blk_dx = g->dx[block];
#define OUT_OF_RANGE(lo, hi)                                                                   \
    if (!((lo) >= nb_begin && (hi) <= nb_end))                                                 \
        return fail(SKO_ERR_RUNTIME, "exchange_block_ghosts: neighbor block cannot supply ghost " \
                                     "width %d", j);
    if (nb_dx == blk_dx) {
        int src = left_side ? iface - j : iface + (j - 1);
        OUT_OF_RANGE(src, src + 1);
        memcpy(ghost, line + (size_t)src * p, sizeof(double) * p);
        return SKO_OK;
    }
    if (nb_dx > blk_dx) {
        int m = (int)llround(nb_dx / blk_dx);
        int coarse = left_side ? iface - 1 - (j - 1) / m : iface + (j - 1) / m;
        OUT_OF_RANGE(coarse, coarse + 1);
        int piece = left_side ? m - 1 - (j - 1) % m : (j - 1) % m;
        double* refined = (double*)malloc(sizeof(double) * (size_t)m * p);
        sko_coarse_to_fine(b, line + (size_t)coarse * p, m, refined);
        memcpy(ghost, refined + (size_t)piece * p, sizeof(double) * p);
        free(refined);
        return SKO_OK;
    }
    int m = (int)llround(blk_dx / nb_dx);
    int lo = left_side ? iface - j * m : iface + (j - 1) * m;
    OUT_OF_RANGE(lo, lo + m);
    sko_fine_to_coarse(b, line + (size_t)lo * p, m, ghost);
    return SKO_OK;
#undef OUT_OF_RANGE
}

/* adaptivity.cpp:211-225 */
int sko_exchange_block_ghosts(const sko_basis* b, const sko_grid* g, int block, const double* line,
                              int gl, int gr, double* ext) {
    const int p = b->p;
    const int cells = g->cells[block];
    const int c0 = g->start[block];
    memcpy(ext + (size_t)gl * p, line + (size_t)c0 * p, sizeof(double) * (size_t)cells * p);
    for (int j = 1; j <= gl; ++j) {
        int rc = fill_ghost(b, g, block, 1, j, line, ext + (size_t)(gl - j) * p);
        if (rc) return rc;
    }
    for (int j = 1; j <= gr; ++j) {
        int rc = fill_ghost(b, g, block, 0, j, line, ext + (size_t)(gl + cells + j - 1) * p);
        if (rc) return rc;
    }
    return SKO_OK;
}

/* advection.cpp:144-207 advect_x */
int sko_advect_x(sko_field* f, double tau, double sqrt_mu, const sko_limiter* lim, int bc,
                 int max_ghost, long step_index, sko_stats* stats) {
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    const int nx = f->x.ncells;
    const sko_grid* grid = &f->x;
    const int nblocks = grid->nblocks;
    if (nblocks > 1 && bc != SKO_BC_ZERO)
        return fail(SKO_ERR_RUNTIME,
                    "advect_x: periodic rule is only supported on single-block grids");
    const int nlines = f->v.ncells * p;
    double* scratch = (double*)malloc(sizeof(double) * (size_t)nx * p);
    double* ext = (double*)malloc(sizeof(double) * (size_t)(nx + 2 * (nx + 2)) * p);
    int rc = SKO_OK;
    sko_stats local = {0};
    for (int lid = 0; lid < nlines && rc == SKO_OK; ++lid) {
        int vc = lid / p, vn = lid % p;
        double speed = sko_v_node(f, vc, vn) / sqrt_mu;
        double* line = f->data + fidx(f, 0, 0, vc, vn);
        if (nblocks == 1) {
            line_plan P;
            make_plan(b, speed, tau, grid->dx[0], lim, &P);
            rc = sko_advect_line(b, P.A, P.B, P.istar, bc, line, 0, nx, 0, scratch,
                                 P.has_lim ? &P.lim : NULL, &local);
        } else {
            for (int bl = 0; bl < nblocks && rc == SKO_OK; ++bl) {
                line_plan P;
                make_plan(b, speed, tau, grid->dx[bl], lim, &P);
                int gl_need = imax2(0, -P.istar);
                int gr_need = imax2(0, P.istar + 1);
                int gl = (bl > 0) ? gl_need : 0;
                int gr = (bl + 1 < nblocks) ? gr_need : 0;
                if (max_ghost >= 0 && imax2(gl, gr) > max_ghost) {
                    g_err_step = step_index;
                    rc = fail(SKO_ERR_SIMULATION,
                              "step %ld: insufficient ghost width: sweep requires %d cells, "
                              "layout provides %d",
                              step_index, imax2(gl, gr), max_ghost);
                    break;
                }
                double* e2 = (double*)malloc(sizeof(double) * (size_t)(gl + grid->cells[bl] + gr) * p);
                rc = sko_exchange_block_ghosts(b, grid, bl, line, gl, gr, e2);
                if (rc == SKO_OK)
                    rc = sko_advect_line(b, P.A, P.B, P.istar, SKO_BC_ZERO, e2, gl,
                                         grid->cells[bl], gr, scratch + (size_t)grid->start[bl] * p,
                                         P.has_lim ? &P.lim : NULL, &local);
                free(e2);
            }
        }
        if (rc == SKO_OK) memcpy(line, scratch, sizeof(double) * (size_t)nx * p);
    }
    free(scratch);
    free(ext);
    if (stats) {
        stats->outputs += local.outputs;
        stats->inline_troubled += local.inline_troubled;
        stats->inline_clamped += local.inline_clamped;
        stats->inline_mean_outside += local.inline_mean_outside;
    }
    return rc;
}

/* advection.cpp:209-238 advect_v */
int sko_advect_v(sko_field* f, double tau, const double* E, double charge_sign, double sqrt_mu,
                 const sko_limiter* lim, int bc, sko_stats* stats) {
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    const int nv = f->v.ncells;
    const int nx = f->x.ncells;
    const double dv = f->v.dx[0];
    const size_t stride = (size_t)nx * p;
    double* in = (double*)malloc(sizeof(double) * (size_t)nv * p);
    double* out = (double*)malloc(sizeof(double) * (size_t)nv * p);
    int rc = SKO_OK;
    for (int lid = 0; lid < nx * p && rc == SKO_OK; ++lid) {
        int xc = lid / p, xn = lid % p;
        double speed = charge_sign * E[(size_t)xc * p + xn] / sqrt_mu;
        line_plan P;
        make_plan(b, speed, tau, dv, lim, &P);
        double* src = f->data + fidx(f, xc, xn, 0, 0);
        for (size_t j = 0; j < (size_t)nv * p; ++j) in[j] = src[j * stride];
        rc = sko_advect_line(b, P.A, P.B, P.istar, bc, in, 0, nv, 0, out,
                             P.has_lim ? &P.lim : NULL, stats);
        for (size_t j = 0; j < (size_t)nv * p; ++j) src[j * stride] = out[j];
    }
    free(in);
    free(out);
    return rc;
}

/* v sweep over pre-gathered lines (used to check the v-sharded halo path):
 * lines are contiguous (gl+n+gr)*p blocks at line_stride doubles. */
int sko_advect_v_lines(const sko_basis* b, int nlines, int line_stride, const double* in, int gl,
                       int n, int gr, double* out, const double* E, double charge_sign,
                       double sqrt_mu, double tau, double dv, const sko_limiter* lim,
                       sko_stats* stats) {
    for (int l = 0; l < nlines; ++l) {
        double speed = charge_sign * E[l] / sqrt_mu;
        line_plan P;
        make_plan(b, speed, tau, dv, lim, &P);
        int rc = sko_advect_line(b, P.A, P.B, P.istar, SKO_BC_ZERO, in + (size_t)l * line_stride,
                                 gl, n, gr, out + (size_t)l * n * b->p,
                                 P.has_lim ? &P.lim : NULL, stats);
        if (rc) return rc;
    }
    return SKO_OK;
}

/* limiters.cpp:254-275 PostPass::run_segment */
static void run_segment(const sko_basis* b, const sko_limiter* cfg, const double* cells, int n,
                        const double* left_nb, const double* right_nb, int wrap, double* out,
                        sko_stats* st) {
    const int p = b->p;
    for (int i = 0; i < n; ++i) {
        const double* t[3];
        for (int d = -1; d <= 1; ++d) {
            int c = i + d;
            const double* ptr;
            if (c >= 0 && c < n)
                ptr = cells + (size_t)c * p;
            else if (wrap)
                ptr = cells + (size_t)(((c % n) + n) % n) * p;
            else if (c < 0)
                ptr = left_nb ? left_nb : kZero;
            else
                ptr = right_nb ? right_nb : kZero;
            t[d + 1] = ptr;
        }
        st->post_checked++;
        int flag = cfg->indicator == SKO_IND_MINMOD
                       ? sko_indicator_minmod(b, t[0], t[1], t[2])
                       : sko_indicator_meanerr(b, t[0], t[1], t[2], cfg->threshold);
        if (flag) {
            st->post_troubled++;
            if (cfg->modifier == SKO_MOD_SIMPLE)
                sko_modify_simple_weno(b, t[0], t[1], t[2], cfg, out + (size_t)i * p);
            else
                sko_modify_line_weno(b, t[0], t[1], t[2], cfg, out + (size_t)i * p);
        } else {
            memcpy(out + (size_t)i * p, t[1], sizeof(double) * p);
        }
    }
}

/* limiters.cpp:280-345 apply_post_limiter; dir 0 = X, 1 = V */
int sko_post_limiter(sko_field* f, int dir, const sko_limiter* cfg, int bc, sko_stats* stats) {
    if (cfg->indicator == SKO_IND_NONE) return SKO_OK;
    if (cfg->modifier == SKO_MOD_LINE && cfg->gamma_line[1] == 0.0)
        return fail(SKO_ERR_RUNTIME, "line WENO: gamma_0 must be nonzero");
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    const int wrap = bc == SKO_BC_PERIODIC;
    const int nx = f->x.ncells, nv = f->v.ncells;
    sko_stats st = {0};
    int rc = SKO_OK;
    if (dir == 0) {
        const sko_grid* g = &f->x;
        if (g->nblocks > 1 && wrap)
            return fail(SKO_ERR_RUNTIME, "apply_post_limiter: periodic rule needs a single-block grid");
        double* scratch = (double*)malloc(sizeof(double) * (size_t)nx * p);
        double* ext = (double*)malloc(sizeof(double) * (size_t)(nx + 2) * p);
        for (int lid = 0; lid < nv * p && rc == SKO_OK; ++lid) {
            double* line = f->data + fidx(f, 0, 0, lid / p, lid % p);
            if (g->nblocks == 1) {
                run_segment(b, cfg, line, nx, NULL, NULL, wrap, scratch, &st);
            } else {
                for (int bl = 0; bl < g->nblocks && rc == SKO_OK; ++bl) {
                    int gl = bl > 0 ? 1 : 0, gr = bl + 1 < g->nblocks ? 1 : 0;
                    rc = sko_exchange_block_ghosts(b, g, bl, line, gl, gr, ext);
                    if (rc) break;
                    run_segment(b, cfg, ext + (size_t)gl * p, g->cells[bl], gl ? ext : NULL,
                                gr ? ext + (size_t)(gl + g->cells[bl]) * p : NULL, 0,
                                scratch + (size_t)g->start[bl] * p, &st);
                }
            }
            if (rc == SKO_OK) memcpy(line, scratch, sizeof(double) * (size_t)nx * p);
        }
        free(scratch);
        free(ext);
    } else {
        const size_t stride = (size_t)nx * p;
        double* in = (double*)malloc(sizeof(double) * (size_t)nv * p);
        double* out = (double*)malloc(sizeof(double) * (size_t)nv * p);
        for (int lid = 0; lid < nx * p; ++lid) {
            double* src = f->data + fidx(f, lid / p, lid % p, 0, 0);
            for (size_t j = 0; j < (size_t)nv * p; ++j) in[j] = src[j * stride];
            run_segment(b, cfg, in, nv, NULL, NULL, wrap, out, &st);
            for (size_t j = 0; j < (size_t)nv * p; ++j) src[j * stride] = out[j];
        }
        free(in);
        free(out);
    }
    if (stats) {
        stats->post_checked += st.post_checked;
        stats->post_troubled += st.post_troubled;
    }
    return rc;
}

/* ======================================================================
 * velocity cut-off  (core/src/adaptivity.cpp:16-130)
 * ==================================================================== */

static int policy_ok(double p, double gamma, double tol) {
    if (!(p > 0 && gamma >= 0 && p + gamma < 1))
        return fail(SKO_ERR_RUNTIME, "VAdjustPolicy: need 0 < p, 0 <= gamma, p + gamma < 1");
    if (!(tol > 0)) return fail(SKO_ERR_RUNTIME, "VAdjustPolicy: tol must be positive");
    return SKO_OK;
}

/* adaptivity.cpp:16-38; returns 1 (shrink), 0 (keep), <0 error */
int sko_check_velocity_shrink(const sko_field* f, double pp, double gamma, double tol) {
    if (policy_ok(pp, gamma, tol)) return -1;
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    const sko_grid* v = &f->v;
    const double dv = v->dx[0];
    const double probe = sko_grid_right(v) * (1.0 - pp - gamma);
    const double signs[2] = {1.0, -1.0};
    for (int s = 0; s < 2; ++s) {
        double vp = signs[s] * probe;
        int vc = (int)floor((vp - v->left[0]) / dv);
        vc = imin2(imax2(vc, 0), v->ncells - 1);
        double xi = (vp - sko_grid_cell_left(v, vc)) / dv;
        double L[SKO_MAXP];
        for (int n = 0; n < p; ++n) L[n] = sko_lagrange(b, n, xi);
        for (int xc = 0; xc < f->x.ncells; ++xc)
            for (int xn = 0; xn < p; ++xn) {
                double val = 0.0;
                for (int vn = 0; vn < p; ++vn) val += L[vn] * f->data[fidx(f, xc, xn, vc, vn)];
                if (fabs(val) >= tol) return 0;
            }
    }
    return 1;
}

typedef struct {
    int old_cell;
    double T[SKO_MAXP * SKO_MAXP];
} vpiece;

/* adaptivity.cpp:94-130 shrink_velocity_domain (+ build_v_transfer :52-90) */
int sko_shrink_velocity_domain(sko_field* f, double pp, double gamma, double tol, double* result) {
    if (policy_ok(pp, gamma, tol)) return SKO_ERR_RUNTIME;
    const sko_basis* b = basis_of(f->k);
    const int p = f->k + 1;
    const int nv = f->v.ncells, nx = f->x.ncells;
    double vmax_before = sko_grid_right(&f->v);
    double mass_before = sko_mass(f);
    double new_vmax = vmax_before * (1.0 - pp);
    sko_grid nv_grid;
    int rc = sko_grid_uniform(&nv_grid, -new_vmax, new_vmax, nv);
    if (rc) return rc;
    /* build_v_transfer */
    const sko_grid* ov = &f->v;
    const double old_dx = ov->dx[0];
    int* npieces = (int*)calloc((size_t)nv, sizeof(int));
    vpiece* pieces = (vpiece*)calloc((size_t)nv * 4, sizeof(vpiece));
    for (int j = 0; j < nv; ++j) {
        double a = sko_grid_cell_left(&nv_grid, j);
        double h = sko_grid_cell_width(&nv_grid, j);
        double bb = a + h;
        int i0 = (int)floor((a - ov->left[0]) / old_dx);
        i0 = imin2(imax2(i0, 0), ov->ncells - 1);
        for (int i = i0; i < ov->ncells; ++i) {
            double oa = sko_grid_cell_left(ov, i), ob = oa + old_dx;
            double s0 = dmax2(a, oa), s1 = dmin2(bb, ob);
            if (s1 <= s0) {
                if (oa >= bb) break;
                continue;
            }
            if (npieces[j] >= 4) {
                free(npieces);
                free(pieces);
                return fail(SKO_ERR_RUNTIME, "shrink: too many overlapping cells");
            }
            vpiece* pc = &pieces[(size_t)j * 4 + npieces[j]++];
            pc->old_cell = i;
            for (int t = 0; t < p * p; ++t) pc->T[t] = 0.0;
            double len = s1 - s0;
            for (int q = 0; q < p; ++q) {
                double x = s0 + len * b->nodes[q];
                double xi_src = (x - oa) / old_dx;
                double xi_tgt = (x - a) / h;
                double wq = b->weights[q] * len;
                for (int m = 0; m < p; ++m) {
                    double lm = sko_lagrange(b, m, xi_tgt) / (b->weights[m] * h);
                    for (int n = 0; n < p; ++n)
                        pc->T[m * p + n] += wq * lm * sko_lagrange(b, n, xi_src);
                }
            }
        }
    }
    const size_t stride = (size_t)nx * p;
    size_t total = (size_t)nx * nv * p * p;
    double* next = (double*)malloc(sizeof(double) * total);
    double* line = (double*)malloc(sizeof(double) * (size_t)nv * p);
    double* out = (double*)malloc(sizeof(double) * (size_t)nv * p);
    for (int xc = 0; xc < nx; ++xc)
        for (int xn = 0; xn < p; ++xn) {
            const double* src0 = f->data + fidx(f, xc, xn, 0, 0);
            for (size_t j = 0; j < (size_t)nv * p; ++j) line[j] = src0[j * stride];
            for (size_t j = 0; j < (size_t)nv * p; ++j) out[j] = 0.0;
            for (int j = 0; j < nv; ++j)
                for (int pi = 0; pi < npieces[j]; ++pi) {
                    const vpiece* pc = &pieces[(size_t)j * 4 + pi];
                    const double* src = line + (size_t)pc->old_cell * p;
                    double* dst = out + (size_t)j * p;
                    for (int m = 0; m < p; ++m) {
                        double acc = 0.0;
                        for (int n = 0; n < p; ++n) acc += pc->T[m * p + n] * src[n];
                        dst[m] += acc;
                    }
                }
            double* dst0 = next + fidx(f, xc, xn, 0, 0);
            for (size_t j = 0; j < (size_t)nv * p; ++j) dst0[j * stride] = out[j];
        }
    memcpy(f->data, next, sizeof(double) * total);
    f->v = nv_grid;
    free(next);
    free(line);
    free(out);
    free(npieces);
    free(pieces);
    if (result) {
        result[0] = vmax_before;
        result[1] = new_vmax;
        result[2] = mass_before;
        result[3] = sko_mass(f);
    }
    return SKO_OK;
}

/* ======================================================================
 * Poisson  (core/src/poisson.cpp)
 * ==================================================================== */

/* poisson.cpp:38-57 ctor */
/* Noise-envelope knob (tests only, tests/golden/make_c3_envelope.py): factor
 * and solve with another LAPACK's dpbtrf_/dpbtrs_ (e.g. the OpenBLAS in the
 * image) instead of the reference-LAPACK restatement. The reference pins no
 * LAPACK (core/CMakeLists.txt:1), so this spread is part of its own noise.
 * Applies to Poisson operators created while it is set. */
static sko_dpbtrf_fn g_lapack_trf = 0;
static sko_dpbtrs_fn g_lapack_trs = 0;
void sko_set_lapack(sko_dpbtrf_fn trf, sko_dpbtrs_fn trs) {
    g_lapack_trf = trf;
    g_lapack_trs = trs;
}

int sko_poisson_init(sko_poisson* P, const sko_grid* g, int k, double penalty_scale) {
    memset(P, 0, sizeof *P);
    if (k < 0) return fail(SKO_ERR_RUNTIME, "PoissonOperator: degree must be >= 0");
    if (!(penalty_scale > 0))
        return fail(SKO_ERR_RUNTIME, "PoissonOperator: penalty_scale must be positive");
    P->grid = *g;
    P->lapack_trs = g_lapack_trs;
    P->k = k;
    P->p = k + 2;
    P->n = g->ncells * (k + 2);
    P->kd = 2 * (k + 2) - 1;
    P->penalty_scale = penalty_scale;
    const sko_basis* bk = basis_of(k);
    const sko_basis* bs = basis_of(k + 1);
    const int ps = P->p;
    for (int m = 0; m < ps; ++m)
        for (int n = 0; n <= k; ++n) P->interp[m * (k + 1) + n] = sko_lagrange(bk, n, bs->nodes[m]);
    for (int m = 0; m <= k; ++m)
        for (int n = 0; n < ps; ++n)
            P->deriv_at_k[m * ps + n] = sko_lagrange_derivative(bs, n, bk->nodes[m]);

    /* poisson.cpp:59-122 assemble */
    const int ldab = P->kd + 1;
    P->band = (double*)calloc((size_t)ldab * P->n, sizeof(double));
#define ADD(i, j, v)                                                   \
    do {                                                               \
        int ii_ = (i), jj_ = (j);                                      \
        if (ii_ >= jj_) P->band[(size_t)jj_ * ldab + (ii_ - jj_)] += (v); \
    } while (0)
    double t0[SKO_MAXP + 1], t1[SKO_MAXP + 1], d0[SKO_MAXP + 1], d1[SKO_MAXP + 1];
    for (int n = 0; n < ps; ++n) {
        t0[n] = sko_lagrange(bs, n, 0.0);
        t1[n] = sko_lagrange(bs, n, 1.0);
        d0[n] = sko_lagrange_derivative(bs, n, 0.0);
        d1[n] = sko_lagrange_derivative(bs, n, 1.0);
    }
    double* M = (double*)malloc(sizeof(double) * 4 * ps * ps);
    for (int c = 0; c < g->ncells; ++c) {
        double h = sko_grid_cell_width(g, c);
        for (int i = 0; i < ps * ps; ++i) M[i] = 0.0;
        for (int q = 0; q < ps; ++q)
            for (int a = 0; a < ps; ++a)
                for (int bb = 0; bb < ps; ++bb)
                    M[a * ps + bb] += bs->weights[q] * bs->diff[q * ps + a] * bs->diff[q * ps + bb] / h;
        for (int a = 0; a < ps; ++a)
            for (int bb = 0; bb < ps; ++bb) ADD(c * ps + a, c * ps + bb, M[a * ps + bb]);
    }
    double pen = penalty_scale * (k + 2) * (k + 2);
    for (int c = 0; c + 1 < g->ncells; ++c) {
        double hl = sko_grid_cell_width(g, c), hr = sko_grid_cell_width(g, c + 1);
        double sigma = pen / dmin2(hl, hr);
        double J[2 * (SKO_MAXP + 1)], D[2 * (SKO_MAXP + 1)];
        for (int n = 0; n < ps; ++n) {
            J[n] = t1[n];
            J[ps + n] = -t0[n];
            D[n] = 0.5 * d1[n] / hl;
            D[ps + n] = 0.5 * d0[n] / hr;
        }
        double defect = 0.0;
        const int w2 = 2 * ps;
        for (int a = 0; a < w2; ++a)
            for (int bb = 0; bb < w2; ++bb) {
                M[a * w2 + bb] = sigma * J[a] * J[bb] - D[a] * J[bb] - J[a] * D[bb];
                if (bb < a) defect = dmax2(defect, fabs(M[a * w2 + bb] - M[bb * w2 + a]));
            }
        P->symmetry_defect = dmax2(P->symmetry_defect, defect);
        for (int a = 0; a < w2; ++a)
            for (int bb = 0; bb < w2; ++bb) ADD(c * ps + a, c * ps + bb, M[a * w2 + bb]);
    }
    {
        double h = sko_grid_cell_width(g, 0);
        double sigma = pen / h;
        for (int a = 0; a < ps; ++a)
            for (int bb = 0; bb < ps; ++bb)
                M[a * ps + bb] = sigma * t0[a] * t0[bb] + d0[a] / h * t0[bb] + t0[a] * d0[bb] / h;
        for (int a = 0; a < ps; ++a)
            for (int bb = 0; bb < ps; ++bb) ADD(a, bb, M[a * ps + bb]);
    }
    {
        int c = g->ncells - 1;
        double h = sko_grid_cell_width(g, c);
        double sigma = pen / h;
        for (int a = 0; a < ps; ++a)
            for (int bb = 0; bb < ps; ++bb)
                M[a * ps + bb] = sigma * t1[a] * t1[bb] - d1[a] / h * t1[bb] - t1[a] * d1[bb] / h;
        for (int a = 0; a < ps; ++a)
            for (int bb = 0; bb < ps; ++bb) ADD(c * ps + a, c * ps + bb, M[a * ps + bb]);
    }
#undef ADD
    free(M);
    /* poisson.cpp:124-133 factorize */
    P->factor = (double*)malloc(sizeof(double) * (size_t)ldab * P->n);
    memcpy(P->factor, P->band, sizeof(double) * (size_t)ldab * P->n);
    int info;
    if (g_lapack_trf) {  /* envelope knob: another LAPACK's dpbtrf_ (Fortran ABI) */
        int n = P->n, kd = P->kd, ld = ldab;
        info = 0;
        g_lapack_trf("L", &n, &kd, P->factor, &ld, &info);
    } else {
        info = sko_dpbtrf_lower(P->n, P->kd, P->factor, ldab);
    }
    if (info != 0)
        return fail(SKO_ERR_RUNTIME,
                    "Poisson factorization failed (matrix not positive definite; penalty_scale "
                    "too small?), dpbtrf info = %d",
                    info);
    return SKO_OK;
}

void sko_poisson_free(sko_poisson* P) {
    free(P->band);
    free(P->factor);
    P->band = P->factor = NULL;
}

/* poisson.cpp:135-149 */
int sko_poisson_build_load(const sko_poisson* P, const double* rho, double* load) {
    const sko_basis* bs = basis_of(P->k + 1);
    const int k = P->k, ps = P->p;
    for (int c = 0; c < P->grid.ncells; ++c) {
        double h = sko_grid_cell_width(&P->grid, c);
        const double* rc = rho + (size_t)c * (k + 1);
        for (int m = 0; m < ps; ++m) {
            double val = 0.0;
            for (int n = 0; n <= k; ++n) val += P->interp[m * (k + 1) + n] * rc[n];
            load[(size_t)c * ps + m] = bs->weights[m] * h * val;
        }
    }
    return SKO_OK;
}

/* poisson.cpp:166-192 solve_raw + solve */
int sko_poisson_solve(const sko_poisson* P, const double* rho, double* phi, double* E) {
    sko_poisson_build_load(P, rho, phi);
    if (P->lapack_trs) {
        int n = P->n, kd = P->kd, ld = P->kd + 1, one = 1, info = 0;
        P->lapack_trs("L", &n, &kd, &one, P->factor, &ld, phi, &n, &info);
    } else {
        sko_dpbtrs_lower(P->n, P->kd, P->factor, P->kd + 1, phi);
    }
    const int k = P->k, ps = P->p;
    for (int c = 0; c < P->grid.ncells; ++c) {
        double h = sko_grid_cell_width(&P->grid, c);
        const double* pc = phi + (size_t)c * ps;
        for (int m = 0; m <= k; ++m) {
            double dphi = 0.0;
            for (int n = 0; n < ps; ++n) dphi += P->deriv_at_k[m * ps + n] * pc[n];
            E[(size_t)c * (k + 1) + m] = -dphi / h;
        }
    }
    return SKO_OK;
}

/* Noise-envelope knob (tests only): 1 = sum electrons before ions in the
 * charge density, a rounding-level perturbation of the reference's order. */
static int g_rho_order = 0;
void sko_set_rho_order(int mode) { g_rho_order = mode; }

/* poisson.cpp:194-216 (ions first, then electrons) */
void sko_charge_density(const sko_field* fe, const sko_field* fi, double* rho) {
    const sko_basis* b = basis_of(fe->k);
    const int p = fe->k + 1;
    const int nx = fe->x.ncells;
    for (int i = 0; i < nx * p; ++i) rho[i] = 0.0;
    const sko_field* fs[2] = {fi, fe};
    double signs[2] = {+1.0, -1.0};
    if (g_rho_order == 1) {
        fs[0] = fe;
        fs[1] = fi;
        signs[0] = -1.0;
        signs[1] = +1.0;
    }
    for (int s = 0; s < 2; ++s) {
        const sko_field* f = fs[s];
        for (int vc = 0; vc < f->v.ncells; ++vc) {
            double dv = sko_grid_cell_width(&f->v, vc);
            for (int vn = 0; vn < p; ++vn) {
                double w = signs[s] * b->weights[vn] * dv;
                for (int xc = 0; xc < nx; ++xc)
                    for (int xn = 0; xn < p; ++xn)
                        rho[(size_t)xc * p + xn] += w * f->data[fidx(f, xc, xn, vc, vn)];
            }
        }
    }
}

/* diagnostics.cpp:71-83 */
double sko_electric_energy(const sko_grid* g, int k, const double* E) {
    const sko_basis* b = basis_of(k);
    const int p = k + 1;
    double acc = 0.0;
    for (int c = 0; c < g->ncells; ++c) {
        double h = sko_grid_cell_width(g, c);
        for (int q = 0; q < p; ++q) {
            double e = E[(size_t)c * p + q];
            acc += 0.5 * b->weights[q] * h * e * e;
        }
    }
    return acc;
}

/* ======================================================================
 * stepper + run loop  (core/src/stepper.cpp:44-103, core/src/run.cpp:26-131)
 * ==================================================================== */

/* run.cpp:19-22 */
static double gaussian_blob(double x, double v, double sigma) {
    return (1.0 / sqrt(2.0 * M_PI)) * exp(-x * x / (2.0 * sigma * sigma)) * exp(-v * v / 2.0);
}

static int field_init(sko_field* f, int species, const sko_grid* x, double vmax, int nv, int k) {
    memset(f, 0, sizeof *f);
    f->species = species;
    f->k = k;
    f->x = *x;
    int rc = sko_grid_uniform(&f->v, -vmax, vmax, nv);
    if (rc) return rc;
    double ext = sko_grid_right(&f->v) - f->v.left[0];
    if (!(fabs(f->v.left[0] + sko_grid_right(&f->v)) <= 1e-12 * ext))
        return fail(SKO_ERR_RUNTIME, "NodalField: v grid must be symmetric about 0");
    size_t n = (size_t)x->ncells * nv * (k + 1) * (k + 1);
    f->data = (double*)calloc(n, sizeof(double));
    return f->data ? SKO_OK : fail(SKO_ERR_RUNTIME, "out of memory");
}

/* field.cpp:42-50 fill with the blob */
static void fill_blob(sko_field* f, double sigma) {
    const int p = f->k + 1;
    for (int vc = 0; vc < f->v.ncells; ++vc)
        for (int vn = 0; vn < p; ++vn) {
            double v = sko_v_node(f, vc, vn);
            for (int xc = 0; xc < f->x.ncells; ++xc)
                for (int xn = 0; xn < p; ++xn)
                    f->data[fidx(f, xc, xn, vc, vn)] = gaussian_blob(sko_x_node(f, xc, xn), v, sigma);
        }
}

int sko_state_init(sko_state* S, double L, double dt, int k, double mu, double sigma, double vmax_e,
                   double vmax_i, int nf, int nc, int m, int nv, const char* limiter,
                   double limiter_threshold, int v_adjust, double adapt_p, double adapt_gamma,
                   double adapt_tol, double penalty_scale) {
    memset(S, 0, sizeof *S);
    if (sigma < 0) sigma = 0.1 * L;
    sko_grid xg;
    int rc = sko_grid_three_block(&xg, -L, L, nf, nc, m);
    if (rc) return rc;
    if ((rc = field_init(&S->fe, 0, &xg, vmax_e, nv, k))) return rc;
    if ((rc = field_init(&S->fi, 1, &xg, vmax_i, nv, k))) return rc;
    fill_blob(&S->fe, sigma);
    fill_blob(&S->fi, sigma);
    S->sigma = sigma;
    S->sqrt_mu_e = 1.0;
    S->charge_e = -1.0;
    if (!(mu > 0)) return fail(SKO_ERR_RUNTIME, "SpeciesParams::ion: mass ratio must be positive");
    S->sqrt_mu_i = sqrt(mu);
    S->charge_i = +1.0;
    S->dt = dt;
    if ((rc = sko_limiter_parse(limiter, &S->limiter))) return rc;
    S->limiter.threshold = limiter_threshold;
    S->bc = SKO_BC_ZERO;
    S->v_adjust = v_adjust;
    S->adapt_p = adapt_p;
    S->adapt_gamma = adapt_gamma;
    S->adapt_tol = adapt_tol;
    S->last_shrink_e = -10;
    S->last_shrink_i = -10;
    if ((rc = sko_poisson_init(&S->poisson, &xg, k, penalty_scale))) return rc;
    size_t nE = (size_t)xg.ncells * (k + 1);
    S->E = (double*)calloc(nE, sizeof(double));
    S->phi = (double*)calloc((size_t)S->poisson.n, sizeof(double));
    double* rho = (double*)calloc(nE, sizeof(double));
    sko_charge_density(&S->fe, &S->fi, rho);
    sko_poisson_solve(&S->poisson, rho, S->phi, S->E);
    free(rho);
    return SKO_OK;
}

/* run.cpp:47-51 source.eval: H(t0 - t) blob(x, v) / t0, H(0) = 1 */
static double source_eval(double t, double x, double v, double t0, double sigma) {
    if (t > t0) return 0.0;
    return gaussian_blob(x, v, sigma) / t0;
}

/* stepper.cpp:29-42; SourceTerm::active (stepper.hpp:19-21): t <= t_end */
void sko_source_half_step(sko_field* f, double t, double half_dt, double t0, double sigma) {
    if (!(t <= t0)) return;
    const int p = f->k + 1;
    for (int vc = 0; vc < f->v.ncells; ++vc)
        for (int vn = 0; vn < p; ++vn) {
            double v = sko_v_node(f, vc, vn);
            for (int xc = 0; xc < f->x.ncells; ++xc)
                for (int xn = 0; xn < p; ++xn) {
                    double x = sko_x_node(f, xc, xn);
                    f->data[fidx(f, xc, xn, vc, vn)] +=
                        0.5 * half_dt * (source_eval(t, x, v, t0, sigma) + source_eval(t + half_dt, x, v, t0, sigma));
                }
        }
}

long sko_state_field_size(sko_state* S, int species);

int sko_state_set_injection(sko_state* S, double t0) {
    if (!(t0 > 0)) return fail(SKO_ERR_RUNTIME, "injection: t0 must be positive");
    S->injection = 1;
    S->t0 = t0;
    memset(S->fe.data, 0, sizeof(double) * (size_t)sko_state_field_size(S, 0));
    memset(S->fi.data, 0, sizeof(double) * (size_t)sko_state_field_size(S, 1));
    size_t nE = (size_t)S->fe.x.ncells * (S->fe.k + 1);
    double* rho = (double*)calloc(nE, sizeof(double));
    sko_charge_density(&S->fe, &S->fi, rho);
    sko_poisson_solve(&S->poisson, rho, S->phi, S->E);
    free(rho);
    return SKO_OK;
}

void sko_state_free(sko_state* S) {
    free(S->fe.data);
    free(S->fi.data);
    free(S->E);
    free(S->phi);
    sko_poisson_free(&S->poisson);
}

/* stepper.cpp:44-103 strang_step */
int sko_strang_step(sko_state* S, int max_ghost) {
    const double dt = S->dt;
    if (dt == 0.0) return fail(SKO_ERR_RUNTIME, "strang_step: dt must be nonzero");
    const double half = 0.5 * dt;
    const sko_limiter* lim = &S->limiter;
    int rc;
    if (S->injection) {
        sko_source_half_step(&S->fe, S->time, half, S->t0, S->sigma);
        sko_source_half_step(&S->fi, S->time, half, S->t0, S->sigma);
    }
#define POST(dir)                                                                  \
    if (lim->indicator != SKO_IND_NONE) {                                          \
        if ((rc = sko_post_limiter(&S->fe, dir, lim, S->bc, &S->stats))) return rc; \
        if ((rc = sko_post_limiter(&S->fi, dir, lim, S->bc, &S->stats))) return rc; \
    }
    if ((rc = sko_advect_x(&S->fe, half, S->sqrt_mu_e, lim, S->bc, max_ghost, S->step, &S->stats)))
        return rc;
    if ((rc = sko_advect_x(&S->fi, half, S->sqrt_mu_i, lim, S->bc, max_ghost, S->step, &S->stats)))
        return rc;
    POST(0);
    {
        size_t nE = (size_t)S->fe.x.ncells * (S->fe.k + 1);
        double* rho = (double*)malloc(sizeof(double) * nE);
        sko_charge_density(&S->fe, &S->fi, rho);
        sko_poisson_solve(&S->poisson, rho, S->phi, S->E);
        free(rho);
    }
    if ((rc = sko_advect_v(&S->fe, dt, S->E, S->charge_e, S->sqrt_mu_e, lim, S->bc, &S->stats)))
        return rc;
    if ((rc = sko_advect_v(&S->fi, dt, S->E, S->charge_i, S->sqrt_mu_i, lim, S->bc, &S->stats)))
        return rc;
    POST(1);
    if ((rc = sko_advect_x(&S->fe, half, S->sqrt_mu_e, lim, S->bc, max_ghost, S->step, &S->stats)))
        return rc;
    if ((rc = sko_advect_x(&S->fi, half, S->sqrt_mu_i, lim, S->bc, max_ghost, S->step, &S->stats)))
        return rc;
    POST(0);
#undef POST
    if (S->injection) {
        sko_source_half_step(&S->fe, S->time + half, half, S->t0, S->sigma);
        sko_source_half_step(&S->fi, S->time + half, half, S->t0, S->sigma);
    }
    S->time += dt;
    S->step += 1;
    if (!sko_all_finite(&S->fe) || !sko_all_finite(&S->fi)) {
        g_err_step = S->step;
        return fail(SKO_ERR_SIMULATION, "step %ld: nonfinite values in the density function",
                    S->step);
    }
    return SKO_OK;
}

/* run.cpp:98-114 check_shrink */
static int check_shrink(sko_state* S, sko_field* f, long* last, int* count) {
    if (!S->v_adjust) return SKO_OK;
    if (S->step - *last < 10) return SKO_OK;
    int c = sko_check_velocity_shrink(f, S->adapt_p, S->adapt_gamma, S->adapt_tol);
    if (c < 0) return SKO_ERR_RUNTIME;
    if (!c) return SKO_OK;
    int rc = sko_shrink_velocity_domain(f, S->adapt_p, S->adapt_gamma, S->adapt_tol, NULL);
    if (rc) return rc;
    *last = S->step;
    ++*count;
    return SKO_OK;
}

/* run.cpp:124-131 loop body */
int sko_run_step(sko_state* S) {
    double vmax_now = dmax2(sko_grid_right(&S->fe.v), sko_grid_right(&S->fi.v));
    double dx_fine = S->fe.x.dx[0];
    double sqrt_mu_min = dmin2(S->sqrt_mu_e, S->sqrt_mu_i);
    int max_ghost = sko_required_ghost_width(vmax_now, S->dt, sqrt_mu_min, dx_fine);
    int rc = sko_strang_step(S, max_ghost);
    if (rc) return rc;
    if ((rc = check_shrink(S, &S->fe, &S->last_shrink_e, &S->shrinks_e))) return rc;
    if ((rc = check_shrink(S, &S->fi, &S->last_shrink_i, &S->shrinks_i))) return rc;
    return SKO_OK;
}

/* ======================================================================
 * opaque-handle accessors for ctypes (mirror oracle/ref_driver.cpp ref_state_*)
 * ==================================================================== */

sko_state* sko_state_new(double L, double dt, int k, double mu, double sigma, double vmax_e,
                         double vmax_i, int nf, int nc, int m, int nv, const char* limiter,
                         double limiter_threshold, int v_adjust, double adapt_p,
                         double adapt_gamma, double adapt_tol, double penalty_scale) {
    sko_state* S = (sko_state*)calloc(1, sizeof(sko_state));
    if (sko_state_init(S, L, dt, k, mu, sigma, vmax_e, vmax_i, nf, nc, m, nv, limiter,
                       limiter_threshold, v_adjust, adapt_p, adapt_gamma, adapt_tol,
                       penalty_scale)) {
        sko_state_free(S);
        free(S);
        return NULL;
    }
    return S;
}
void sko_state_delete(sko_state* S) {
    if (!S) return;
    sko_state_free(S);
    free(S);
}
static sko_field* sfield(sko_state* S, int species) { return species == 0 ? &S->fe : &S->fi; }
double* sko_state_field(sko_state* S, int species) { return sfield(S, species)->data; }
long sko_state_field_size(sko_state* S, int species) {
    sko_field* f = sfield(S, species);
    return (long)f->x.ncells * f->v.ncells * (f->k + 1) * (f->k + 1);
}
double sko_state_vmax(sko_state* S, int species) { return sko_grid_right(&sfield(S, species)->v); }
double* sko_state_E(sko_state* S) { return S->E; }
/* tests only: the Poisson load vector (poisson.cpp:135-149) */
int sko_state_poisson_load(sko_state* S, const double* rho, double* load) {
    return sko_poisson_build_load(&S->poisson, rho, load);
}
/* tests only: the assembled SIPG band before factorisation, (kd+1) x n column-major lower */
const double* sko_state_poisson_band(sko_state* S, int* n, int* kd) {
    *n = S->poisson.n;
    *kd = S->poisson.kd;
    return S->poisson.band;
}
double* sko_state_phi(sko_state* S) { return S->phi; }
long sko_state_step_index(sko_state* S) { return S->step; }
int sko_state_shrinks(sko_state* S, int species) {
    return species == 0 ? S->shrinks_e : S->shrinks_i;
}
long sko_state_last_shrink(sko_state* S, int species) {
    return species == 0 ? S->last_shrink_e : S->last_shrink_i;
}
void sko_state_stats(sko_state* S, long* out) {
    out[0] = S->stats.outputs;
    out[1] = S->stats.inline_troubled;
    out[2] = S->stats.inline_clamped;
    out[3] = S->stats.inline_mean_outside;
    out[4] = S->stats.post_checked;
    out[5] = S->stats.post_troubled;
}
int sko_state_advect_x(sko_state* S, int species, double tau, int limited, int max_ghost) {
    sko_limiter none;
    sko_limiter_parse("none", &none);
    return sko_advect_x(sfield(S, species), tau, species == 0 ? S->sqrt_mu_e : S->sqrt_mu_i,
                        limited ? &S->limiter : &none, S->bc, max_ghost, S->step, &S->stats);
}
int sko_state_advect_v(sko_state* S, int species, double tau, const double* E, int limited) {
    sko_limiter none;
    sko_limiter_parse("none", &none);
    return sko_advect_v(sfield(S, species), tau, E, species == 0 ? S->charge_e : S->charge_i,
                        species == 0 ? S->sqrt_mu_e : S->sqrt_mu_i, limited ? &S->limiter : &none,
                        S->bc, &S->stats);
}
int sko_state_post_limit(sko_state* S, int species, int dir, const char* mode) {
    sko_limiter cfg;
    int rc = sko_limiter_parse(mode, &cfg);
    if (rc) return rc;
    return sko_post_limiter(sfield(S, species), dir, &cfg, S->bc, &S->stats);
}
void sko_state_charge_density(sko_state* S, double* rho) { sko_charge_density(&S->fe, &S->fi, rho); }
int sko_state_poisson_solve(sko_state* S, const double* rho, double* E, double* phi) {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)S->poisson.n);
    int rc = sko_poisson_solve(&S->poisson, rho, tmp, E);
    if (phi) memcpy(phi, tmp, sizeof(double) * (size_t)S->poisson.n);
    free(tmp);
    return rc;
}
int sko_state_check_shrink(sko_state* S, int species) {
    return sko_check_velocity_shrink(sfield(S, species), S->adapt_p, S->adapt_gamma, S->adapt_tol);
}
int sko_state_shrink(sko_state* S, int species, double* result) {
    return sko_shrink_velocity_domain(sfield(S, species), S->adapt_p, S->adapt_gamma, S->adapt_tol,
                                      result);
}
/* mass_e, mass_i, l2_e, l2_i, e_energy, vmax_e, vmax_i, mom_e, mom_i, ekin_e, ekin_i */
void sko_state_summary(sko_state* S, double* out) {
    out[0] = sko_mass(&S->fe);
    out[1] = sko_mass(&S->fi);
    out[2] = sko_l2_norm(&S->fe);
    out[3] = sko_l2_norm(&S->fi);
    out[4] = sko_electric_energy(&S->fe.x, S->fe.k, S->E);
    out[5] = sko_grid_right(&S->fe.v);
    out[6] = sko_grid_right(&S->fi.v);
    out[7] = sko_momentum(&S->fe);
    out[8] = sko_momentum(&S->fi);
    out[9] = sko_kinetic_energy(&S->fe);
    out[10] = sko_kinetic_energy(&S->fi);
}

/* One x line of advect_x (advection.cpp:160-201) for a given speed: used to
 * check sampled lines of full-size GPU sweeps without a full CPU field. */
int sko_advect_x_line(int k, int nblocks, const double* left, const int* cells, const double* dx,
                      double speed, double tau, int inline_sldg, double threshold, int max_ghost,
                      const double* line, double* out) {
    const sko_basis* b = basis_of(k);
    const int p = k + 1;
    sko_grid g;
    int rc = sko_grid_init(&g, nblocks, left, cells, dx);
    if (rc) return rc;
    sko_limiter lim;
    sko_limiter_parse(inline_sldg ? "sldg" : "none", &lim);
    lim.threshold = threshold;
    sko_stats st = {0};
    for (int bl = 0; bl < g.nblocks; ++bl) {
        line_plan P;
        make_plan(b, speed, tau, g.dx[bl], &lim, &P);
        int gl = bl > 0 ? imax2(0, -P.istar) : 0;
        int gr = bl + 1 < g.nblocks ? imax2(0, P.istar + 1) : 0;
        if (g.nblocks == 1) gl = gr = 0;
        if (max_ghost >= 0 && imax2(gl, gr) > max_ghost)
            return fail(SKO_ERR_SIMULATION, "insufficient ghost width");
        double* e2 = (double*)malloc(sizeof(double) * (size_t)(gl + g.cells[bl] + gr) * p);
        rc = sko_exchange_block_ghosts(b, &g, bl, line, gl, gr, e2);
        if (rc == SKO_OK)
            rc = sko_advect_line(b, P.A, P.B, P.istar, SKO_BC_ZERO, e2, gl, g.cells[bl], gr,
                                 out + (size_t)g.start[bl] * p, P.has_lim ? &P.lim : NULL, &st);
        free(e2);
        if (rc) return rc;
    }
    return SKO_OK;
}
