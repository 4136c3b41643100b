// sk_host.cpp -- host-side setup numerics of the B200 sLdG library.
//
// * reference-cell constants with the reference's formulas and operation order
//   (core/src/basis.cpp:14-91) so device tables derived from them are bitwise
//   equal to the reference's;
// * block-structured grid bookkeeping (core/src/grid.cpp:9-62);
// * the SIPG Poisson band assembled as in core/src/poisson.cpp:59-122, then
//   reduced once by block cyclic reduction into a plan the device replays each
//   step (replaces the serial LAPACK dpbtrf/dpbtrs pair, poisson.cpp:124-174).
#include <cmath>
#include <cstring>
#include <string>

#include "sk_internal.hpp"

namespace sk {

namespace {

void legendre_wd(int n, double t, double& P, double& dP) {  // basis.cpp:14-25
    double p0 = 1.0, p1 = t;
    if (n == 0) {
        P = 1.0;
        dP = 0.0;
        return;
    }
    for (int j = 2; j <= n; ++j) {
        double p2 = ((2 * j - 1) * t * p1 - (j - 1) * p0) / j;
        p0 = p1;
        p1 = p2;
    }
    P = p1;
    dP = n * (t * p1 - p0) / (t * t - 1.0);
}

}  // namespace

Basis make_basis(int k) {  // basis.cpp:29-91
    Basis b;
    std::memset(&b, 0, sizeof b);
    b.k = k;
    b.p = k + 1;
    const int n = k + 1;
    for (int i = 0; i < n; ++i) {
        double t = -std::cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int iter = 0; iter < 100; ++iter) {
            double P, dP;
            legendre_wd(n, t, P, dP);
            double dt = P / dP;
            t -= dt;
            if (std::abs(dt) < 1e-15) break;
        }
        double P, dP;
        legendre_wd(n, t, P, dP);
        b.nodes[i] = 0.5 * (t + 1.0);
        b.weights[i] = 1.0 / ((1.0 - t * t) * dP * dP);
    }
    const int p = n;
    for (int i = 0; i < p; ++i) {
        b.bary[i] = 1.0;
        for (int j = 0; j < p; ++j)
            if (j != i) b.bary[i] /= (b.nodes[i] - b.nodes[j]);
    }
    for (int m = 0; m < p; ++m) {
        double row_sum = 0.0;
        for (int n2 = 0; n2 < p; ++n2) {
            if (n2 == m) continue;
            double d = b.bary[n2] / b.bary[m] / (b.nodes[m] - b.nodes[n2]);
            b.diff[m * p + n2] = d;
            row_sum += d;
        }
        b.diff[m * p + m] = -row_sum;
    }
    for (int n2 = 0; n2 < p; ++n2) {
        double c[SK_MAXP] = {};
        c[0] = b.bary[n2];
        int deg = 0;
        for (int j = 0; j < p; ++j) {
            if (j == n2) continue;
            for (int d = deg; d >= 0; --d) {
                c[d + 1] += c[d];
                c[d] *= -b.nodes[j];
            }
            ++deg;
        }
        for (int d = 0; d < p; ++d) b.mono[d * p + n2] = c[d];
    }
    for (int j = 0; j < 33; ++j) b.cheb[j] = std::cos(M_PI * (2 * j + 1) / 66.0);
    // evaluate() terms at the cell ends (sk_numerics.cuh EvalPt): same
    // division and ordered sum as evaluate() performs at run time
    b.ev0den = 0.0;
    b.ev1den = 0.0;
    for (int n = 0; n < p; ++n) {
        b.ev0[n] = b.bary[n] / (0.0 - b.nodes[n]);
        b.ev1[n] = b.bary[n] / (1.0 - b.nodes[n]);
    }
    for (int n = 0; n < p; ++n) {
        b.ev0den += b.ev0[n];
        b.ev1den += b.ev1[n];
    }
    return b;
}

double host_lagrange(const Basis& b, int n, double xi) {
    double v = b.bary[n];
    for (int j = 0; j < b.p; ++j)
        if (j != n) v *= (xi - b.nodes[j]);
    return v;
}

double host_lagrange_derivative(const Basis& b, int n, double xi) {  // basis.cpp:110-121
    double acc = 0.0;
    for (int j = 0; j < b.p; ++j) {
        if (j == n) continue;
        double term = 1.0;
        for (int i = 0; i < b.p; ++i)
            if (i != n && i != j) term *= (xi - b.nodes[i]);
        acc += term;
    }
    return b.bary[n] * acc;
}

// ---------------- grid (grid.cpp) ----------------
std::string grid_init(Grid& g, int nblocks, const double* left, const int* cells, const double* dx) {
    g = Grid{};
    if (nblocks < 1) return "Grid1D: needs at least one block";
    if (nblocks > kMaxBlocks) return "Grid1D: too many blocks";
    g.nblocks = nblocks;
    for (int b = 0; b < nblocks; ++b) {
        if (!(cells[b] >= 1 && dx[b] > 0)) return "Grid1D: block must have cells >= 1, dx > 0";
        if (b > 0) {
            double prev_right = left[b - 1] + cells[b - 1] * dx[b - 1];
            if (!(std::abs(prev_right - left[b]) <= 1e-12 * (std::abs(left[b]) + dx[b - 1])))
                return "Grid1D: blocks must be contiguous";
            double coarse = dmax2(dx[b - 1], dx[b]);
            double fine = dmin2(dx[b - 1], dx[b]);
            double ratio = coarse / fine;
            if (!(std::abs(ratio - std::round(ratio)) < 1e-10 && std::round(ratio) >= 1))
                return "Grid1D: adjacent block widths must satisfy dx_coarse = m * dx_fine";
        }
        g.left[b] = left[b];
        g.cells[b] = cells[b];
        g.dx[b] = dx[b];
        g.ncells += cells[b];
        g.start[b + 1] = g.ncells;
        int c = -1;
        for (int i = 0; i < g.nclass; ++i)
            if (g.class_dx[i] == dx[b]) c = i;
        if (c < 0) {
            c = g.nclass++;
            g.class_dx[c] = dx[b];
        }
        g.cls[b] = c;
    }
    return "";
}

int grid_block_of(const Grid& g, int cell) {
    for (int b = 0; b < g.nblocks; ++b)
        if (cell < g.start[b + 1]) return b;
    return g.nblocks - 1;
}
double grid_cell_left(const Grid& g, int cell) {
    int b = grid_block_of(g, cell);
    return g.left[b] + (cell - g.start[b]) * g.dx[b];
}
double grid_cell_width(const Grid& g, int cell) { return g.dx[grid_block_of(g, cell)]; }
double grid_right(const Grid& g) {
    int b = g.nblocks - 1;
    return g.left[b] + g.cells[b] * g.dx[b];
}

// ---------------- Poisson ----------------
namespace {

using Mat = std::vector<double>;

Mat matmul(const Mat& A, const Mat& B, int p) {
    Mat C(p * p, 0.0);
    for (int i = 0; i < p; ++i)
        for (int k = 0; k < p; ++k) {
            double a = A[i * p + k];
            for (int j = 0; j < p; ++j) C[i * p + j] += a * B[k * p + j];
        }
    return C;
}

bool invert(const Mat& A, Mat& inv, int p) {  // Gauss-Jordan, partial pivoting
    Mat M = A;
    inv.assign(p * p, 0.0);
    for (int i = 0; i < p; ++i) inv[i * p + i] = 1.0;
    for (int c = 0; c < p; ++c) {
        int piv = c;
        for (int r = c + 1; r < p; ++r)
            if (std::abs(M[r * p + c]) > std::abs(M[piv * p + c])) piv = r;
        if (M[piv * p + c] == 0.0) return false;
        if (piv != c)
            for (int j = 0; j < p; ++j) {
                std::swap(M[c * p + j], M[piv * p + j]);
                std::swap(inv[c * p + j], inv[piv * p + j]);
            }
        double d = M[c * p + c];
        for (int j = 0; j < p; ++j) {
            M[c * p + j] /= d;
            inv[c * p + j] /= d;
        }
        for (int r = 0; r < p; ++r) {
            if (r == c) continue;
            double f = M[r * p + c];
            if (f == 0.0) continue;
            for (int j = 0; j < p; ++j) {
                M[r * p + j] -= f * M[c * p + j];
                inv[r * p + j] -= f * inv[c * p + j];
            }
        }
    }
    return true;
}

}  // namespace

std::string poisson_plan_build(PoissonPlan& P, const Grid& g, int k, double penalty_scale) {
    if (k < 0) return "PoissonOperator: degree must be >= 0";
    if (!(penalty_scale > 0)) return "PoissonOperator: penalty_scale must be positive";
    const Basis bk = make_basis(k);
    const Basis bs = make_basis(k + 1);
    const int ps = k + 2;
    const int N = g.ncells;
    const int n = N * ps;
    const int kd = 2 * ps - 1;
    const int ldab = kd + 1;
    P = PoissonPlan{};
    P.k = k;
    P.ps = ps;
    P.ncells = N;
    P.interp.assign(ps * (k + 1), 0.0);
    for (int m = 0; m < ps; ++m)
        for (int nn = 0; nn <= k; ++nn) P.interp[m * (k + 1) + nn] = host_lagrange(bk, nn, bs.nodes[m]);
    P.deriv.assign((k + 1) * ps, 0.0);
    for (int m = 0; m <= k; ++m)
        for (int nn = 0; nn < ps; ++nn)
            P.deriv[m * ps + nn] = host_lagrange_derivative(bs, nn, bk.nodes[m]);
    P.h.resize(N);
    for (int c = 0; c < N; ++c) P.h[c] = grid_cell_width(g, c);
    P.ws.assign(bs.weights, bs.weights + ps);

    // --- assemble exactly as poisson.cpp:59-122 ---
    std::vector<double>& band = P.band;
    band.assign(size_t(ldab) * n, 0.0);
    auto add = [&](int i, int j, double v) {
        if (i >= j) band[size_t(j) * ldab + (i - j)] += v;
    };
    std::vector<double> t0(ps), t1(ps), d0(ps), d1(ps);
    for (int nn = 0; nn < ps; ++nn) {
        t0[nn] = host_lagrange(bs, nn, 0.0);
        t1[nn] = host_lagrange(bs, nn, 1.0);
        d0[nn] = host_lagrange_derivative(bs, nn, 0.0);
        d1[nn] = host_lagrange_derivative(bs, nn, 1.0);
    }
    for (int c = 0; c < N; ++c) {
        double h = grid_cell_width(g, c);
        std::vector<double> vol(ps * ps, 0.0);
        for (int q = 0; q < ps; ++q)
            for (int a = 0; a < ps; ++a)
                for (int b2 = 0; b2 < ps; ++b2)
                    vol[a * ps + b2] += bs.weights[q] * bs.diff[q * ps + a] * bs.diff[q * ps + b2] / h;
        for (int a = 0; a < ps; ++a)
            for (int b2 = 0; b2 < ps; ++b2) add(c * ps + a, c * ps + b2, vol[a * ps + b2]);
    }
    double pen = penalty_scale * (k + 2) * (k + 2);
    for (int c = 0; c + 1 < N; ++c) {
        double hl = grid_cell_width(g, c), hr = grid_cell_width(g, c + 1);
        double sigma = pen / dmin2(hl, hr);
        std::vector<double> J(2 * ps), D(2 * ps);
        for (int nn = 0; nn < ps; ++nn) {
            J[nn] = t1[nn];
            J[ps + nn] = -t0[nn];
            D[nn] = 0.5 * d1[nn] / hl;
            D[ps + nn] = 0.5 * d0[nn] / hr;
        }
        const int w2 = 2 * ps;
        std::vector<double> M(w2 * w2);
        for (int a = 0; a < w2; ++a)
            for (int b2 = 0; b2 < w2; ++b2) {
                M[a * w2 + b2] = sigma * J[a] * J[b2] - D[a] * J[b2] - J[a] * D[b2];
                if (b2 < a)
                    P.symmetry_defect = dmax2(P.symmetry_defect, std::abs(M[a * w2 + b2] - M[b2 * w2 + a]));
            }
        for (int a = 0; a < w2; ++a)
            for (int b2 = 0; b2 < w2; ++b2) add(c * ps + a, c * ps + b2, M[a * w2 + b2]);
    }
    {
        double h = grid_cell_width(g, 0), sigma = pen / h;
        for (int a = 0; a < ps; ++a)
            for (int b2 = 0; b2 < ps; ++b2)
                add(a, b2, sigma * t0[a] * t0[b2] + d0[a] / h * t0[b2] + t0[a] * d0[b2] / h);
    }
    {
        int c = N - 1;
        double h = grid_cell_width(g, c), sigma = pen / h;
        for (int a = 0; a < ps; ++a)
            for (int b2 = 0; b2 < ps; ++b2)
                add(c * ps + a, c * ps + b2,
                    sigma * t1[a] * t1[b2] - d1[a] / h * t1[b2] - t1[a] * d1[b2] / h);
    }

    // --- reference-LAPACK dpbtf2 factor (poisson.cpp:124-133), for the
    //     exact-reduction mode that replays dpbtrs on the device ---
    P.kd = kd;
    P.chol = band;
    for (int j = 0; j < n; ++j) {
        double* col = P.chol.data() + (size_t)j * ldab;
        double ajj = col[0];
        if (ajj <= 0.0) return "Poisson factorization failed (matrix not positive definite)";
        ajj = std::sqrt(ajj);
        col[0] = ajj;
        const int kn = kd < n - 1 - j ? kd : n - 1 - j;
        if (kn > 0) {
            const double r = 1.0 / ajj;
            for (int i = 1; i <= kn; ++i) col[i] = r * col[i];
            for (int jj = 0; jj < kn; ++jj) {
                const double xj = col[1 + jj];
                if (xj != 0.0) {
                    const double temp = -1.0 * xj;
                    double* c2 = P.chol.data() + (size_t)(j + 1 + jj) * ldab;
                    for (int ii = jj; ii < kn; ++ii) c2[ii - jj] = c2[ii - jj] + col[1 + ii] * temp;
                }
            }
        }
    }

    // --- block tridiagonal view of the band ---
    auto full = [&](int r, int c) -> double {
        if (r < c) std::swap(r, c);
        if (r - c > kd) return 0.0;
        return band[size_t(c) * ldab + (r - c)];
    };
    const int pp = ps * ps;
    std::vector<Mat> D(N, Mat(pp)), Lo(N, Mat(pp, 0.0)), Up(N, Mat(pp, 0.0));
    for (int q = 0; q < N; ++q)
        for (int a = 0; a < ps; ++a)
            for (int b2 = 0; b2 < ps; ++b2) {
                D[q][a * ps + b2] = full(q * ps + a, q * ps + b2);
                if (q > 0) Lo[q][a * ps + b2] = full(q * ps + a, (q - 1) * ps + b2);
                if (q + 1 < N) Up[q][a * ps + b2] = full(q * ps + a, (q + 1) * ps + b2);
            }

    // --- block cyclic reduction (even positions survive each level) ---
    int Nl = N;
    long off = 0, koff = 0, ooff = 0;
    auto put_t = [&](std::vector<double>& dst, long base, int rows, int r, const Mat& M) {
        // [ps*ps][rows] block starting at base*pp
        for (int e = 0; e < pp; ++e) dst[(size_t)base * pp + (size_t)e * rows + r] = M[e];
    };
    while (true) {
        const int Nn = (Nl + 1) / 2, No = Nl / 2;
        P.level_n.push_back(Nl);
        P.level_off.push_back(off);
        P.keep_off.push_back(koff);
        P.odd_off.push_back(ooff);
        std::vector<Mat> Dinv(Nl);
        for (int q = 0; q < Nl; ++q)
            if (!invert(D[q], Dinv[q], ps))
                return "Poisson factorization failed (singular block in cyclic reduction)";
        if (Nl == 1) {
            P.DinvTop = Dinv[0];
            break;
        }
        P.LoT.resize((size_t)(ooff + No) * pp);
        P.UpT.resize((size_t)(ooff + No) * pp);
        P.DinvT.resize((size_t)(ooff + No) * pp);
        for (int o = 0; o < No; ++o) {
            const int q = 2 * o + 1;
            put_t(P.LoT, ooff, No, o, Lo[q]);
            put_t(P.UpT, ooff, No, o, Up[q]);
            put_t(P.DinvT, ooff, No, o, Dinv[q]);
        }
        P.AlphaT.resize((size_t)(koff + Nn) * pp, 0.0);
        P.GammaT.resize((size_t)(koff + Nn) * pp, 0.0);
        std::vector<Mat> D2(Nn), Lo2(Nn, Mat(pp, 0.0)), Up2(Nn, Mat(pp, 0.0));
        for (int r = 0; r < Nn; ++r) {
            int q = 2 * r;
            Mat Dn = D[q];
            Mat alpha(pp, 0.0), gamma(pp, 0.0);
            if (q - 1 >= 0) {
                alpha = matmul(Lo[q], Dinv[q - 1], ps);
                for (auto& v : alpha) v = -v;
                Mat t = matmul(alpha, Up[q - 1], ps);
                for (int i = 0; i < pp; ++i) Dn[i] += t[i];
                Lo2[r] = matmul(alpha, Lo[q - 1], ps);
            }
            if (q + 1 < Nl) {
                gamma = matmul(Up[q], Dinv[q + 1], ps);
                for (auto& v : gamma) v = -v;
                Mat t = matmul(gamma, Lo[q + 1], ps);
                for (int i = 0; i < pp; ++i) Dn[i] += t[i];
                Up2[r] = matmul(gamma, Up[q + 1], ps);
            }
            // symmetrise the Schur complement against roundoff drift
            for (int a = 0; a < ps; ++a)
                for (int b2 = a + 1; b2 < ps; ++b2) {
                    double sm = 0.5 * (Dn[a * ps + b2] + Dn[b2 * ps + a]);
                    Dn[a * ps + b2] = Dn[b2 * ps + a] = sm;
                }
            D2[r] = Dn;
            put_t(P.AlphaT, koff, Nn, r, alpha);
            put_t(P.GammaT, koff, Nn, r, gamma);
        }
        off += Nl;
        koff += Nn;
        ooff += No;
        D.swap(D2);
        Lo.swap(Lo2);
        Up.swap(Up2);
        Nl = Nn;
    }
    P.nlevels = (int)P.level_n.size();
    return "";
}

}  // namespace sk
