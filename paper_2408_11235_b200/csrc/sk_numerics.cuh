// sk_numerics.cuh -- per-cell sLdG arithmetic for sm_100a (device + host).
//
// Every function keeps the reference's floating-point operation order so the
// kernels (compiled with -fmad=false, see build.py) reproduce the reference
// bit for bit given the same inputs:
//   lagrange / evaluate / mean / moments / extrema   core/src/basis.cpp:102-225
//   decompose_shift / shift matrices                 core/src/advection.cpp:14-66
//   inline sLdG limiter                              core/src/limiters.cpp:167-222
//   post-limiter indicators / WENO modifiers         core/src/limiters.cpp:47-165
//   coarse<->fine transfer                           core/src/adaptivity.cpp:132-156
// P = k+1 is a template parameter so every loop unrolls into registers.
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#define SK_HD __host__ __device__ __forceinline__
#define SK_MAXP 8

namespace sk {

// Reference-cell constants, computed once on the host with the reference's
// formulas (sk_host.cpp) and passed by value in kernel parameter space.
struct Basis {
    int k, p;
    double nodes[SK_MAXP];
    double weights[SK_MAXP];
    double bary[SK_MAXP];
    double mono[SK_MAXP * SK_MAXP];  // nodal -> monomial, row-major [d][n]
    double diff[SK_MAXP * SK_MAXP];  // nodal differentiation [m][n]
    double cheb[33];                 // cos(pi(2j+1)/66), basis.cpp:211 (k > 3)
    // evaluate() at xi = 0 and xi = 1 (basis.cpp:123-134): the barycentric
    // terms t_n = bary[n] / (xi - x_n) and their ordered sum, computed once
    double ev0[SK_MAXP], ev0den;
    double ev1[SK_MAXP], ev1den;
};

SK_HD double dmax2(double a, double b) { return (a < b) ? b : a; }  // std::max
SK_HD double dmin2(double a, double b) { return (b < a) ? b : a; }  // std::min

// basis.cpp:102-108
template <int P>
SK_HD double lagrange(const Basis& b, int n, double xi) {
    double v = b.bary[n];
#pragma unroll
    for (int j = 0; j < P; ++j)
        if (j != n) v *= (xi - b.nodes[j]);
    return v;
}

// basis.cpp:123-134 (second barycentric form, exact at nodes)
template <int P>
SK_HD double evaluate(const Basis& b, const double* u, double xi) {
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
        if (xi == b.nodes[n]) return u[n];
        double t = b.bary[n] / (xi - b.nodes[n]);
        num += t * u[n];
        den += t;
    }
    return num / den;
}

// basis.cpp:136-140
template <int P>
SK_HD double mean(const Basis& b, const double* u) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < P; ++j) acc += b.weights[j] * u[j];
    return acc;
}

// basis.cpp:142-150
template <int P>
SK_HD double integrate(const Basis& b, const double* u, double a, double bb) {
    double acc = 0.0;
    const double len = bb - a;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        double xi = a + len * b.nodes[q];
        acc += b.weights[q] * evaluate<P>(b, u, xi);
    }
    return acc * len;
}

// basis.cpp:152-161
template <int P>
SK_HD void interval_moments(const Basis& b, double a, double bb, double* m) {
    const double len = bb - a;
#pragma unroll
    for (int n = 0; n < P; ++n) m[n] = 0.0;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        double xi = a + len * b.nodes[q];
#pragma unroll
        for (int n = 0; n < P; ++n) m[n] += b.weights[q] * len * lagrange<P>(b, n, xi);
    }
}

// basis.cpp:172-215 extremum_on; IS_MAX selects the comparison.
template <int P, bool IS_MAX>
SK_HD bool better(double x, double y) { return IS_MAX ? (x > y) : (x < y); }

template <int P, bool IS_MAX>
SK_HD double extremum_on(const Basis& b, const double* u, double a, double bb) {
    double best = evaluate<P>(b, u, a);
    if (bb == a) return best;
    double vb = evaluate<P>(b, u, bb);
    if (better<P, IS_MAX>(vb, best)) best = vb;
    if constexpr (P <= 2) {
        return best;
    } else if constexpr (P <= 4) {
        double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < P; ++d) {  // basis.cpp:163-170 to_monomial
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < P; ++n) acc += b.mono[d * P + n] * u[n];
            c[d] = acc;
        }
        double qa = 3.0 * c[3], qb = 2.0 * c[2], qc = c[1];
        double x0 = 0.0, x1 = 0.0;
        int nc = 0;
        if (fabs(qa) > 0.0) {
            double disc = qb * qb - 4.0 * qa * qc;
            if (disc >= 0.0) {
                double r = sqrt(disc);
                x0 = (-qb + r) / (2.0 * qa);
                x1 = (-qb - r) / (2.0 * qa);
                nc = 2;
            }
        } else if (fabs(qb) > 0.0) {
            x0 = -qc / qb;
            nc = 1;
        }
        if (nc >= 1 && x0 > a && x0 < bb) {
            double v = evaluate<P>(b, u, x0);
            if (better<P, IS_MAX>(v, best)) best = v;
        }
        if (nc >= 2 && x1 > a && x1 < bb) {
            double v = evaluate<P>(b, u, x1);
            if (better<P, IS_MAX>(v, best)) best = v;
        }
        return best;
    } else {
        for (int j = 0; j < 33; ++j) {
            double x = 0.5 * (a + bb) + 0.5 * (bb - a) * b.cheb[j];
            double v = evaluate<P>(b, u, x);
            if (better<P, IS_MAX>(v, best)) best = v;
        }
        return best;
    }
}

// evaluate(u, xi) at a point fixed for many u: the barycentric terms are
// computed once; same operations in the same order as evaluate(), so the
// value is bitwise evaluate()'s. hit >= 0: xi is node `hit` (exact return).
template <int P>
struct EvalPt {
    double t[P];
    double den;
    int hit;
};
template <int P>
SK_HD EvalPt<P> make_evalpt(const Basis& b, double xi) {
    EvalPt<P> e;
    e.hit = -1;
    e.den = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
        if (e.hit < 0 && xi == b.nodes[n]) e.hit = n;
        e.t[n] = b.bary[n] / (xi - b.nodes[n]);
    }
    if (e.hit < 0) {
#pragma unroll
        for (int n = 0; n < P; ++n) e.den += e.t[n];
    }
    return e;
}
template <int P>
SK_HD EvalPt<P> basis_evalpt(const Basis& b, int one) {  // xi = 0 or 1 (never a GL node)
    EvalPt<P> e;
    e.hit = -1;
#pragma unroll
    for (int n = 0; n < P; ++n) e.t[n] = one ? b.ev1[n] : b.ev0[n];
    e.den = one ? b.ev1den : b.ev0den;
    return e;
}
template <int P>
SK_HD double eval_at(const EvalPt<P>& e, const double* u) {
    if (e.hit >= 0) return u[e.hit];
    double num = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) num += e.t[n] * u[n];
    return num / e.den;
}

// extremum_on<P,true> and extremum_on<P,false> of the same (u, [a, bb]) in one
// pass: both visit the same candidate points with the same values and differ
// only in the comparison, so (mx, mn) are bitwise the two separate results.
template <int P>
SK_HD void extremum_minmax(const Basis& b, const double* u, double a, double bb, const EvalPt<P>& pa,
                           const EvalPt<P>& pb, double& mx, double& mn) {
    const double va = eval_at<P>(pa, u);
    mx = va;
    mn = va;
    if (bb == a) return;
    const double vb = eval_at<P>(pb, u);
    if (vb > mx) mx = vb;
    if (vb < mn) mn = vb;
    if constexpr (P <= 2) {
        return;
    } else if constexpr (P <= 4) {
        double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < P; ++d) {  // basis.cpp:163-170 to_monomial
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < P; ++n) acc += b.mono[d * P + n] * u[n];
            c[d] = acc;
        }
        double qa = 3.0 * c[3], qb = 2.0 * c[2], qc = c[1];
        double x0 = 0.0, x1 = 0.0;
        int nc = 0;
        if (fabs(qa) > 0.0) {
            double disc = qb * qb - 4.0 * qa * qc;
            if (disc >= 0.0) {
                double r = sqrt(disc);
                x0 = (-qb + r) / (2.0 * qa);
                x1 = (-qb - r) / (2.0 * qa);
                nc = 2;
            }
        } else if (fabs(qb) > 0.0) {
            x0 = -qc / qb;
            nc = 1;
        }
        if (nc >= 1 && x0 > a && x0 < bb) {
            const double v = evaluate<P>(b, u, x0);
            if (v > mx) mx = v;
            if (v < mn) mn = v;
        }
        if (nc >= 2 && x1 > a && x1 < bb) {
            const double v = evaluate<P>(b, u, x1);
            if (v > mx) mx = v;
            if (v < mn) mn = v;
        }
    } else {
        for (int j = 0; j < 33; ++j) {
            const double x = 0.5 * (a + bb) + 0.5 * (bb - a) * b.cheb[j];
            const double v = evaluate<P>(b, u, x);
            if (v > mx) mx = v;
            if (v < mn) mn = v;
        }
    }
}

// advection.cpp:14-25
SK_HD void decompose_shift(double speed, double dt, double dx, int& istar, double& alpha) {
    double s = -speed * dt / dx;
    double fl = floor(s);
    double al = s - fl;
    int is = (int)fl;
    if (al >= 1.0) {
        al -= 1.0;
        is += 1;
    }
    istar = is;
    alpha = al;
}

// advection.cpp:27-66 (alpha in [0,1) by construction of decompose_shift)
template <int P>
SK_HD void shift_matrices(const Basis& b, double alpha, double* A, double* B) {
#pragma unroll
    for (int i = 0; i < P * P; ++i) {
        A[i] = 0.0;
        B[i] = 0.0;
    }
    const double len_a = 1.0 - alpha;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        double xi = len_a * b.nodes[q];
#pragma unroll
        for (int m = 0; m < P; ++m) {
            double lm = lagrange<P>(b, m, xi);
#pragma unroll
            for (int n = 0; n < P; ++n)
                A[m * P + n] += b.weights[q] * len_a * lagrange<P>(b, n, xi + alpha) * lm;
        }
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
        double xi = 1.0 - alpha + alpha * b.nodes[q];
#pragma unroll
        for (int m = 0; m < P; ++m) {
            double lm = lagrange<P>(b, m, xi);
#pragma unroll
            for (int n = 0; n < P; ++n)
                B[m * P + n] += b.weights[q] * alpha * lagrange<P>(b, n, alpha * b.nodes[q]) * lm;
        }
    }
#pragma unroll
    for (int m = 0; m < P; ++m) {
        double inv_w = 1.0 / b.weights[m];
#pragma unroll
        for (int n = 0; n < P; ++n) {
            A[m * P + n] *= inv_w;
            B[m * P + n] *= inv_w;
        }
    }
}

// Fast-mode arithmetic: the same sums contracted into DFMA (acc += a*b as one
// rounding). Used only when the context is not in exact mode; the north-star
// tolerance (1e-12 relative) bounds its effect, the exact mode keeps the
// reference's rounding sequence (-fmad=false everywhere else).
template <bool FMA>
SK_HD double madd(double acc, double a, double b) {
    if constexpr (FMA)
        return fma(a, b, acc);
    else
        return acc + a * b;
}
template <int P, bool FMA>
SK_HD double mean_f(const Basis& b, const double* u) {
    if constexpr (!FMA) {
        return mean<P>(b, u);
    } else {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) acc = fma(b.weights[j], u[j], acc);
        return acc;
    }
}
// one output node: reference acc += A*ul + B*ur (j ascending), or two DFMA
template <int P, bool FMA>
SK_HD double project_node(const double* am, const double* bm, const double* ul, const double* ur) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < P; ++j) {
        if constexpr (FMA)
            acc = fma(bm[j], ur[j], fma(am[j], ul[j], acc));
        else
            acc += am[j] * ul[j] + bm[j] * ur[j];
    }
    return acc;
}
template <int P, bool FMA>
SK_HD void project_cell_f(const double* A, const double* B, const double* ul, const double* ur,
                          double* o) {
#pragma unroll
    for (int m = 0; m < P; ++m) o[m] = project_node<P, FMA>(A + m * P, B + m * P, ul, ur);
}

// advection.cpp:95-101: acc += A*ul + B*ur, j ascending
template <int P>
SK_HD void project_cell(const double* A, const double* B, const double* ul, const double* ur,
                        double* o) {
#pragma unroll
    for (int m = 0; m < P; ++m) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) acc += A[m * P + j] * ul[j] + B[m * P + j] * ur[j];
        o[m] = acc;
    }
}

// Inline sLdG limiter indicator, limiters.cpp:175-189 (cheap: runs on every cell).
template <int P>
SK_HD bool inline_indicator(const Basis& b, double threshold, const double* ext_l,
                            const double* ext_r, const double* ul, const double* ur,
                            const double* up) {
    double mean_l = mean<P>(b, ul);
    double mean_r = mean<P>(b, ur);
    double denom = dmax2(fabs(mean_l), fabs(mean_r));
    if (denom <= 0.0) return false;
    double el = 0.0, er = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
        el += ext_l[n] * up[n];
        er += ext_r[n] * up[n];
    }
    double ind = (fabs(el - mean_l) + fabs(er - mean_r)) / denom;
    return ind > threshold;
}

// `num / den > thr` (limiters.cpp:178-188) decided without the division when
// that is provably the same answer. With thr in [2^-60, 2^60], den in
// [2^-900, 2^900) and hi = RN(thr(1+2^-50)), lo = RN(thr(1-2^-50)):
//   num > RN(hi*den)  =>  num/den > thr(1+2^-51)  =>  RN(num/den) > thr,
//   num < RN(lo*den)  =>  num/den < thr           =>  RN(num/den) <= thr,
// so only the ~2^-50-wide band around the threshold (and NaN, zero or
// out-of-range operands) pays for the correctly rounded quotient.
struct ThrCut {
    double thr, hi, lo;
};
SK_HD ThrCut make_thr_cut(double thr) {
    ThrCut t{thr, HUGE_VAL, -HUGE_VAL};  // +-inf: always the exact path
    if (thr >= 0x1p-60 && thr <= 0x1p60) {
        t.hi = thr * (1.0 + 0x1p-50);
        t.lo = thr * (1.0 - 0x1p-50);
    }
    return t;
}
SK_HD bool over_threshold(double num, double den, const ThrCut& t) {
#ifdef __CUDA_ARCH__
    const unsigned e = (unsigned)__double2hiint(den) - 0x07b00000u;  // den in [2^-900, 2^900)
    if (e < 0x78300000u - 0x07b00000u) {
        const bool up = num > t.hi * den;
        if (up || num < t.lo * den) return up;
    }
#endif
    if (!(den > 0.0)) return false;
    return num / den > t.thr;
}

// inline_indicator with the source-cell means supplied by the caller (a sweep
// that walks cells in order reuses the right mean as the next left one)
template <int P, bool FMA = false>
SK_HD bool inline_indicator_m(const ThrCut& t, const double* ext_l, const double* ext_r,
                              double mean_l, double mean_r, const double* up) {
    double denom = dmax2(fabs(mean_l), fabs(mean_r));
    double el = 0.0, er = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
        el = madd<FMA>(el, ext_l[n], up[n]);
        er = madd<FMA>(er, ext_r[n], up[n]);
    }
    return over_threshold(fabs(el - mean_l) + fabs(er - mean_r), denom, t);
}

// theta clamp of a troubled cell, limiters.cpp:191-215. Returns flags:
// bit0 troubled, bit1 clamped, bit2 mean_outside; `up` modified in place.
template <int P>
SK_HD int inline_clamp(const Basis& b, double alpha, const double* ul, const double* ur,
                       double* up) {
    int flags = 1;
    double mean_p = mean<P>(b, up);
    // the six extremum_on calls of limiters.cpp:196-201 as three min/max pairs
    const EvalPt<P> pa = make_evalpt<P>(b, alpha), p0 = basis_evalpt<P>(b, 0), p1 = basis_evalpt<P>(b, 1);
    double lmax, lmin, rmax, rmin, pmax, pmin;
    extremum_minmax<P>(b, ul, alpha, 1.0, pa, p1, lmax, lmin);
    extremum_minmax<P>(b, ur, 0.0, alpha, p0, pa, rmax, rmin);
    extremum_minmax<P>(b, up, 0.0, 1.0, p0, p1, pmax, pmin);
    double wmax = dmax2(lmax, rmax);
    double wmin = dmin2(lmin, rmin);
    if ((mean_p > wmax) || (mean_p < wmin)) flags |= 4;
    double theta = 1.0;
    double dmx = pmax - mean_p;
    if (dmx != 0.0) theta = dmin2(theta, fabs((wmax - mean_p) / dmx));
    double dmn = pmin - mean_p;
    if (dmn != 0.0) theta = dmin2(theta, fabs((wmin - mean_p) / dmn));
    if (theta < 1.0) {
#pragma unroll
        for (int j = 0; j < P; ++j) up[j] = theta * (up[j] - mean_p) + mean_p;
        flags |= 2;
    }
    return flags;
}

// Fast-mode clamp (k <= 3): the same candidate points (interval ends and the
// interior roots of p'), but every value comes from Horner's rule on the
// monomial coefficients the root search needs anyway -- no barycentric
// divisions. Agrees with inline_clamp to rounding (tolerance mode only).
template <int P>
SK_HD void extremum_minmax_fast(const Basis& b, const double* u, double a, double bb, double& mx,
                                double& mn) {
    static_assert(P <= 4, "fast extremum search is for k <= 3");
    double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int d = 0; d < P; ++d) {
        double acc = 0.0;
#pragma unroll
        for (int n = 0; n < P; ++n) acc = fma(b.mono[d * P + n], u[n], acc);
        c[d] = acc;
    }
    auto horner = [&](double x) { return fma(fma(fma(c[3], x, c[2]), x, c[1]), x, c[0]); };
    const double va = horner(a);
    mx = va;
    mn = va;
    if (bb == a) return;
    const double vb = horner(bb);
    mx = fmax(mx, vb);
    mn = fmin(mn, vb);
    if constexpr (P >= 3) {
        const double qa = 3.0 * c[3], qb = 2.0 * c[2], qc = c[1];
        double x0 = 0.0, x1 = 0.0;
        int nc = 0;
        if (fabs(qa) > 0.0) {
            const double disc = qb * qb - 4.0 * qa * qc;
            if (disc >= 0.0) {
                const double r = sqrt(disc), inv = 1.0 / (2.0 * qa);
                x0 = (-qb + r) * inv;
                x1 = (-qb - r) * inv;
                nc = 2;
            }
        } else if (fabs(qb) > 0.0) {
            x0 = -qc / qb;
            nc = 1;
        }
        if (nc >= 1 && x0 > a && x0 < bb) {
            const double v = horner(x0);
            mx = fmax(mx, v);
            mn = fmin(mn, v);
        }
        if (nc >= 2 && x1 > a && x1 < bb) {
            const double v = horner(x1);
            mx = fmax(mx, v);
            mn = fmin(mn, v);
        }
    }
}

template <int P, bool FMA>
SK_HD int inline_clamp_f(const Basis& b, double alpha, const double* ul, const double* ur, double* up) {
    if constexpr (!FMA || P > 4) {
        return inline_clamp<P>(b, alpha, ul, ur, up);
    } else {
        int flags = 1;
        const double mean_p = mean_f<P, true>(b, up);
        double lmax, lmin, rmax, rmin, pmax, pmin;
        extremum_minmax_fast<P>(b, ul, alpha, 1.0, lmax, lmin);
        extremum_minmax_fast<P>(b, ur, 0.0, alpha, rmax, rmin);
        extremum_minmax_fast<P>(b, up, 0.0, 1.0, pmax, pmin);
        const double wmax = dmax2(lmax, rmax), wmin = dmin2(lmin, rmin);
        if ((mean_p > wmax) || (mean_p < wmin)) flags |= 4;
        double theta = 1.0;
        const double dmx = pmax - mean_p;
        if (dmx != 0.0) theta = dmin2(theta, fabs((wmax - mean_p) / dmx));
        const double dmn = pmin - mean_p;
        if (dmn != 0.0) theta = dmin2(theta, fabs((wmin - mean_p) / dmn));
        if (theta < 1.0) {
#pragma unroll
            for (int j = 0; j < P; ++j) up[j] = fma(theta, up[j] - mean_p, mean_p);
            flags |= 2;
        }
        return flags;
    }
}

// Inline sLdG limiter, limiters.cpp:217-222 (indicator, then clamp).
template <int P>
SK_HD int inline_limit(const Basis& b, double alpha, double threshold, const double* ext_l,
                       const double* ext_r, const double* ul, const double* ur, double* up) {
    if (!inline_indicator<P>(b, threshold, ext_l, ext_r, ul, ur, up)) return 0;
    return inline_clamp<P>(b, alpha, ul, ur, up);
}

// ---------------- post limiters (limiters.cpp:47-165) ----------------
SK_HD double minmod(double a, double b, double c) {
    // branch-free, same values: one of the three sign cases is selected
    const double mpos = dmin2(a, dmin2(b, c));
    const double mneg = -dmin2(-a, dmin2(-b, -c));
    const bool pos = (a > 0) & (b > 0) & (c > 0);
    const bool neg = (a < 0) & (b < 0) & (c < 0);
    return pos ? mpos : (neg ? mneg : 0.0);
}

template <int P>
SK_HD bool indicator_minmod(const Basis& b, const double* um, const double* u0, const double* up) {
    double mean_m = mean<P>(b, um);
    double mean_0 = mean<P>(b, u0);
    double mean_p = mean<P>(b, up);
    double u0_plus = evaluate<P>(b, u0, 1.0) - mean_0;
    double u0_minus = mean_0 - evaluate<P>(b, u0, 0.0);
    double d_plus = mean_p - mean_0;
    double d_minus = mean_0 - mean_m;
    double scale = fabs(mean_m);
    double v;
    v = fabs(mean_0); if (scale < v) scale = v;
    v = fabs(mean_p); if (scale < v) scale = v;
    v = fabs(u0_plus); if (scale < v) scale = v;
    v = fabs(u0_minus); if (scale < v) scale = v;
    v = fabs(d_plus); if (scale < v) scale = v;
    v = fabs(d_minus); if (scale < v) scale = v;
    double guard = 1e-13 * scale;
    return fabs(minmod(u0_plus, d_plus, d_minus) - u0_plus) > guard ||
           fabs(minmod(u0_minus, d_plus, d_minus) - u0_minus) > guard;
}

template <int P>
SK_HD bool indicator_meanerr(const Basis& b, const double* um, const double* u0, const double* up,
                             double threshold) {
    double mean_m = mean<P>(b, um);
    double mean_0 = mean<P>(b, u0);
    double mean_p = mean<P>(b, up);
    double denom = dmax2(fabs(mean_m), dmax2(fabs(mean_0), fabs(mean_p)));
    if (denom <= 0.0) return false;
    double ext_m = integrate<P>(b, um, 1.0, 2.0);
    double ext_p = integrate<P>(b, up, -1.0, 0.0);
    double ind = (fabs(ext_m - mean_0) + fabs(ext_p - mean_0)) / denom;
    return ind > threshold;
}

template <int P>
SK_HD double smoothness_beta(const Basis& b, const double* u) {
    double cur[P], nxt[P];
#pragma unroll
    for (int i = 0; i < P; ++i) cur[i] = u[i];
    double total = 0.0;
#pragma unroll
    for (int s = 1; s < P; ++s) {
#pragma unroll
        for (int m = 0; m < P; ++m) {
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < P; ++n) acc += b.diff[m * P + n] * cur[n];
            nxt[m] = acc;
        }
#pragma unroll
        for (int q = 0; q < P; ++q) total += b.weights[q] * nxt[q] * nxt[q];
#pragma unroll
        for (int i = 0; i < P; ++i) cur[i] = nxt[i];
    }
    return total;
}

struct PostCfg {
    int indicator;  // 1 minmod, 2 meanerr
    int modifier;   // 1 simple WENO, 2 line WENO
    double threshold;
    double gamma_simple[3];
    double gamma_line[3];
    double epsilon;
    // evaluate() at the quadrature points of integrate(u, 1, 2) (ip) and of
    // integrate(u, -1, 0) (im), basis.cpp:142-150: barycentric terms and
    // their ordered sums, computed once on the host with evaluate()'s
    // operations (the points never coincide with a node)
    double ipt[SK_MAXP][SK_MAXP], ipden[SK_MAXP];
    double imt[SK_MAXP][SK_MAXP], imden[SK_MAXP];
    // fast mode: reciprocals of the denominators (and of evaluate()'s at 0, 1)
    double iprc[SK_MAXP], imrc[SK_MAXP], ev0rc, ev1rc;
    // fast mode, mean error: each extension integral as one linear functional
    // of the cell's nodes, sum_q w_q t[q][n] / den[q] folded on the host
    double ipw[SK_MAXP], imw[SK_MAXP];
    // fast mode, simple WENO: the neighbours' polynomials at this cell's nodes,
    // evaluate(u, 1 + xi_m) = sum_n evm[m][n] u[n] and evaluate(u, xi_m - 1) =
    // sum_n evp[m][n] u[n] (the barycentric weights at fixed points, host)
    double evm[SK_MAXP][SK_MAXP], evp[SK_MAXP][SK_MAXP];
    double rg0;  // 1 / gamma_line[1]
};

// host: fill PostCfg's evaluation points for a basis
inline void post_cfg_points(const Basis& b, PostCfg& c) {
    for (int side = 0; side < 2; ++side) {
        const double a = side == 0 ? 1.0 : -1.0, len = (side == 0 ? 2.0 : 0.0) - a;
        for (int q = 0; q < b.p; ++q) {
            const double xi = a + len * b.nodes[q];
            double den = 0.0;
            for (int n = 0; n < b.p; ++n) {
                const double t = b.bary[n] / (xi - b.nodes[n]);
                (side == 0 ? c.ipt : c.imt)[q][n] = t;
                den += t;
            }
            (side == 0 ? c.ipden : c.imden)[q] = den;
            (side == 0 ? c.iprc : c.imrc)[q] = 1.0 / den;
        }
    }
    c.ev0rc = 1.0 / b.ev0den;
    c.ev1rc = 1.0 / b.ev1den;
    for (int n = 0; n < b.p; ++n) {
        double wp = 0.0, wm = 0.0;
        for (int q = 0; q < b.p; ++q) {
            wp += b.weights[q] * c.ipt[q][n] / c.ipden[q];
            wm += b.weights[q] * c.imt[q][n] / c.imden[q];
        }
        c.ipw[n] = wp;
        c.imw[n] = wm;
    }
    for (int m = 0; m < b.p; ++m)
        for (int side = 0; side < 2; ++side) {
            const double xi = side == 0 ? 1.0 + b.nodes[m] : b.nodes[m] - 1.0;
            double den = 0.0, t[SK_MAXP];
            for (int n = 0; n < b.p; ++n) {
                t[n] = b.bary[n] / (xi - b.nodes[n]);  // (xi is never a node: |xi| > 1 off [0, 1])
                den += t[n];
            }
            for (int n = 0; n < b.p; ++n) (side == 0 ? c.evm : c.evp)[m][n] = t[n] / den;
        }
    c.rg0 = 1.0 / c.gamma_line[1];
}

// integrate(u, 1, 2) / integrate(u, -1, 0) with the precomputed points:
// bitwise integrate<P>(b, u, a, a + 1)
template <int P>
SK_HD double integrate_pre(const Basis& b, const double (*t)[SK_MAXP], const double* den, const double* u) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        double num = 0.0;
#pragma unroll
        for (int n = 0; n < P; ++n) num += t[q][n] * u[n];
        acc += b.weights[q] * (num / den[q]);
    }
    return acc * 1.0;
}

// fast-mode indicators (tolerance mode): DFMA sums and multiplication by the
// precomputed reciprocals instead of the exact-order divisions
template <int P>
SK_HD double eval_end_fast(const Basis& b, const double* u, int one, double rc) {
    double num = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) num = fma(one ? b.ev1[n] : b.ev0[n], u[n], num);
    return num * rc;
}
// The post-limiter indicators split into a per-cell summary and a decision
// from the three summaries of a stencil: indicator_minmod / indicator_meanerr
// above with PostCfg's precomputed points (fast mode: DFMA sums, the
// reciprocals, each mean-error extension folded into one functional), the
// same operations in the same order wherever a cell is met, so a pass that
// meets every cell once (the flags fused into the sweeps) decides bitwise
// like the stencil passes.
// minmod: (mean, value at xi = 1, value at xi = 0); meanerr: (mean, the cell's
// extension over its right neighbour, over its left neighbour).
struct PostSum {
    double m, a, b;
};
template <int P, bool FAST, int IND>
SK_HD PostSum post_summary(const Basis& b, const PostCfg& c, const double* u) {
    PostSum s;
    if constexpr (FAST) {
        s.m = mean_f<P, true>(b, u);
        if constexpr (IND == 1) {
            s.a = eval_end_fast<P>(b, u, 1, c.ev1rc);
            s.b = eval_end_fast<P>(b, u, 0, c.ev0rc);
        } else {
            double ea = 0.0, eb = 0.0;
#pragma unroll
            for (int n = 0; n < P; ++n) {
                ea = fma(c.ipw[n], u[n], ea);
                eb = fma(c.imw[n], u[n], eb);
            }
            s.a = ea;
            s.b = eb;
        }
    } else {
        s.m = mean<P>(b, u);
        if constexpr (IND == 1) {
            s.a = eval_at<P>(basis_evalpt<P>(b, 1), u);
            s.b = eval_at<P>(basis_evalpt<P>(b, 0), u);
        } else {
            s.a = integrate_pre<P>(b, c.ipt, c.ipden, u);
            s.b = integrate_pre<P>(b, c.imt, c.imden, u);
        }
    }
    return s;
}
template <bool FAST, int IND>
SK_HD bool post_decide(const PostCfg& c, const PostSum& sm, const PostSum& s0, const PostSum& sp) {
    if constexpr (IND == 1) {  // minmod
        const double u0_plus = s0.a - s0.m;
        const double u0_minus = s0.m - s0.b;
        const double d_plus = sp.m - s0.m;
        const double d_minus = s0.m - sm.m;
        if constexpr (FAST) {
            // |minmod(a, d+, d-) - a| without forming minmod: |a| - min(|a|, |d+|, |d-|) when all
            // three share a sign (the same rounding: fl(mn - |a|) = -fl(|a| - mn)), else |a|;
            // the slopes' part is common to both ends
            const double mbc = fmin(fabs(d_plus), fabs(d_minus));
            const bool pos = (d_plus > 0) & (d_minus > 0), neg = (d_plus < 0) & (d_minus < 0);
            auto dev = [&](double a) {
                const double aa = fabs(a);
                return ((pos & (a > 0)) | (neg & (a < 0))) ? aa - fmin(aa, mbc) : aa;
            };
            const double dp = dev(u0_plus), dm = dev(u0_minus);
            if (!(dp > 0.0) && !(dm > 0.0)) return false;  // (a zero deviation never exceeds the guard)
            const double scale = fmax(fmax(fmax(fabs(sm.m), fabs(s0.m)), fmax(fabs(sp.m), fabs(u0_plus))),
                                      fmax(fmax(fabs(u0_minus), fabs(d_plus)), fabs(d_minus)));
            const double guard = 1e-13 * scale;
            return (dp > guard) | (dm > guard);
        } else {
            double scale = fabs(sm.m);
            double v;
            v = fabs(s0.m); if (scale < v) scale = v;
            v = fabs(sp.m); if (scale < v) scale = v;
            v = fabs(u0_plus); if (scale < v) scale = v;
            v = fabs(u0_minus); if (scale < v) scale = v;
            v = fabs(d_plus); if (scale < v) scale = v;
            v = fabs(d_minus); if (scale < v) scale = v;
            const double guard = 1e-13 * scale;
            return fabs(minmod(u0_plus, d_plus, d_minus) - u0_plus) > guard ||
                   fabs(minmod(u0_minus, d_plus, d_minus) - u0_minus) > guard;
        }
    } else {  // mean error: ext_m = sm.a, ext_p = sp.b
        if constexpr (FAST) {
            const double denom = fmax(fabs(sm.m), fmax(fabs(s0.m), fabs(sp.m)));
            if (!(denom > 0.0)) return false;
            return fabs(sm.a - s0.m) + fabs(sp.b - s0.m) > c.threshold * denom;
        } else {
            const double denom = dmax2(fabs(sm.m), dmax2(fabs(s0.m), fabs(sp.m)));
            if (denom <= 0.0) return false;
            const double ind = (fabs(sm.a - s0.m) + fabs(sp.b - s0.m)) / denom;
            return ind > c.threshold;
        }
    }
}
template <int P, bool FAST, int IND>
SK_HD bool post_flag_sum(const Basis& b, const PostCfg& c, const double* um, const double* u0, const double* up) {
    return post_decide<FAST, IND>(c, post_summary<P, FAST, IND>(b, c, um), post_summary<P, FAST, IND>(b, c, u0),
                                  post_summary<P, FAST, IND>(b, c, up));
}

template <int P>
SK_HD void modify_simple_weno(const Basis& b, const double* um, const double* u0, const double* up,
                              const PostCfg& cfg, double* out) {
    double beta_m = smoothness_beta<P>(b, um);
    double beta_0 = smoothness_beta<P>(b, u0);
    double beta_p = smoothness_beta<P>(b, up);
    const double eps = cfg.epsilon;
    double wm = cfg.gamma_simple[0] / ((eps + beta_m) * (eps + beta_m));
    double w0 = cfg.gamma_simple[1] / ((eps + beta_0) * (eps + beta_0));
    double wp = cfg.gamma_simple[2] / ((eps + beta_p) * (eps + beta_p));
    double sum = wm + w0 + wp;
    wm /= sum;
    w0 /= sum;
    wp /= sum;
    double mean_0 = mean<P>(b, u0);
    double ext_mean_m = integrate<P>(b, um, 1.0, 2.0);
    double ext_mean_p = integrate<P>(b, up, -1.0, 0.0);
#pragma unroll
    for (int m = 0; m < P; ++m) {
        double xi = b.nodes[m];
        double cand_m = evaluate<P>(b, um, 1.0 + xi) - ext_mean_m + mean_0;
        double cand_p = evaluate<P>(b, up, xi - 1.0) - ext_mean_p + mean_0;
        out[m] = wm * cand_m + w0 * u0[m] + wp * cand_p;
    }
}

// fast mode (tolerance): the same modification with the fixed-point
// evaluations and extension integrals as precomputed linear functionals and
// one reciprocal for the weight normalisation -- 4 divisions instead of ~90
template <int P>
SK_HD void modify_simple_weno_fast(const Basis& b, const double* um, const double* u0, const double* up,
                                   const PostCfg& cfg, double* out) {
    const double beta_m = smoothness_beta<P>(b, um);
    const double beta_0 = smoothness_beta<P>(b, u0);
    const double beta_p = smoothness_beta<P>(b, up);
    const double eps = cfg.epsilon;
    double wm = cfg.gamma_simple[0] / ((eps + beta_m) * (eps + beta_m));
    double w0 = cfg.gamma_simple[1] / ((eps + beta_0) * (eps + beta_0));
    double wp = cfg.gamma_simple[2] / ((eps + beta_p) * (eps + beta_p));
    const double rs = 1.0 / (wm + w0 + wp);
    wm *= rs;
    w0 *= rs;
    wp *= rs;
    const double mean_0 = mean_f<P, true>(b, u0);
    double ext_m = 0.0, ext_p = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
        ext_m = fma(cfg.ipw[n], um[n], ext_m);
        ext_p = fma(cfg.imw[n], up[n], ext_p);
    }
#pragma unroll
    for (int m = 0; m < P; ++m) {
        double em = 0.0, ep = 0.0;
#pragma unroll
        for (int n = 0; n < P; ++n) {
            em = fma(cfg.evm[m][n], um[n], em);
            ep = fma(cfg.evp[m][n], up[n], ep);
        }
        const double cand_m = em - ext_m + mean_0;
        const double cand_p = ep - ext_p + mean_0;
        out[m] = fma(wm, cand_m, fma(w0, u0[m], wp * cand_p));
    }
}

template <int P>
SK_HD void modify_line_weno(const Basis& b, const double* um, const double* u0, const double* up,
                            const PostCfg& cfg, double* out) {
    double mean_m = mean<P>(b, um);
    double mean_0 = mean<P>(b, u0);
    double mean_p = mean<P>(b, up);
    double bm = mean_0 - mean_m, am = mean_0 - 0.5 * bm;
    double bp = mean_p - mean_0, ap = mean_0 - 0.5 * bp;
    const double gm = cfg.gamma_line[0], g0 = cfg.gamma_line[1], gp = cfg.gamma_line[2];
    double pm[P], pp[P], p0[P];
#pragma unroll
    for (int m = 0; m < P; ++m) {
        double xi = b.nodes[m];
        pm[m] = am + bm * xi;
        pp[m] = ap + bp * xi;
        p0[m] = (u0[m] - gm * pm[m] - gp * pp[m]) / g0;
    }
    double beta_m = smoothness_beta<P>(b, um);
    double beta_0 = smoothness_beta<P>(b, u0);
    double beta_p = smoothness_beta<P>(b, up);
    double tau = 0.5 * (fabs(beta_0 - beta_m) + fabs(beta_0 - beta_p));
    tau *= tau;
    const double eps = cfg.epsilon;
    double wm = gm * (1.0 + tau / (eps + beta_m));
    double w0 = g0 * (1.0 + tau / (eps + beta_0));
    double wp = gp * (1.0 + tau / (eps + beta_p));
    double sum = wm + w0 + wp;
    wm /= sum;
    w0 /= sum;
    wp /= sum;
#pragma unroll
    for (int m = 0; m < P; ++m) out[m] = wm * pm[m] + w0 * p0[m] + wp * pp[m];
}

template <int P>
SK_HD void modify_line_weno_fast(const Basis& b, const double* um, const double* u0, const double* up,
                                 const PostCfg& cfg, double* out) {
    const double mean_m = mean_f<P, true>(b, um);
    const double mean_0 = mean_f<P, true>(b, u0);
    const double mean_p = mean_f<P, true>(b, up);
    const double bm = mean_0 - mean_m, am = mean_0 - 0.5 * bm;
    const double bp = mean_p - mean_0, ap = mean_0 - 0.5 * bp;
    const double gm = cfg.gamma_line[0], g0 = cfg.gamma_line[1], gp = cfg.gamma_line[2];
    double pm[P], pp[P], p0[P];
#pragma unroll
    for (int m = 0; m < P; ++m) {
        const double xi = b.nodes[m];
        pm[m] = fma(bm, xi, am);
        pp[m] = fma(bp, xi, ap);
        p0[m] = (u0[m] - gm * pm[m] - gp * pp[m]) * cfg.rg0;
    }
    const double beta_m = smoothness_beta<P>(b, um);
    const double beta_0 = smoothness_beta<P>(b, u0);
    const double beta_p = smoothness_beta<P>(b, up);
    double tau = 0.5 * (fabs(beta_0 - beta_m) + fabs(beta_0 - beta_p));
    tau *= tau;
    const double eps = cfg.epsilon;
    double wm = gm * (1.0 + tau / (eps + beta_m));
    double w0 = g0 * (1.0 + tau / (eps + beta_0));
    double wp = gp * (1.0 + tau / (eps + beta_p));
    const double rs = 1.0 / (wm + w0 + wp);
    wm *= rs;
    w0 *= rs;
    wp *= rs;
#pragma unroll
    for (int m = 0; m < P; ++m) out[m] = fma(wm, pm[m], fma(w0, p0[m], wp * pp[m]));
}

// ---------------- sheath-mesh transfer (adaptivity.cpp:132-156) ----------------
// (MC > 0: the refinement ratio m == MC known at compile time, so the loops
// unroll and every load issues up front -- same operations, same order)
// coarse_to_fine, one piece, one node: evaluate(coarse, (piece + x_q)/m)
template <int P, int MC = 0>
SK_HD double coarse_to_fine_node(const Basis& b, const double* coarse, int m, int piece, int q) {
    if constexpr (MC > 0) m = MC;
    return evaluate<P>(b, coarse, (piece + b.nodes[q]) / m);
}

// fine_to_coarse, output node mm, from m consecutive fine cells (stride P)
template <int P, int MC = 0>
SK_HD double fine_to_coarse_node(const Basis& b, const double* fine, int m, int mm) {
    if constexpr (MC > 0) m = MC;
    double acc = 0.0;
#pragma unroll (MC > 0 ? MC : 1)
    for (int j = 0; j < m; ++j) {
        const double* cell = fine + j * P;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            double xi_c = (j + b.nodes[q]) / m;
            acc += b.weights[q] / m * cell[q] * lagrange<P>(b, mm, xi_c);
        }
    }
    return acc / b.weights[mm];
}

}  // namespace sk
