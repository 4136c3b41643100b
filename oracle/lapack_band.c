/*
 * lapack_band.c -- CPU ORACLE (test infrastructure only).
 *
 * The reference factors and solves its SIPG Poisson band with LAPACK
 * dpbtrf_/dpbtrs_ (core/src/poisson.cpp:9-14,128,171); it pins no LAPACK
 * version (core/CMakeLists.txt:1). LAPACK is absent from /root/reference, so
 * this file restates the published reference-LAPACK 3.x algorithm:
 *   dpbtrf('L') with kd < nb(=32)  ->  unblocked dpbtf2:
 *       ajj = sqrt(ab(1,j)); dscal(kn, 1/ajj, ab(2,j)); dsyr('L', kn, -1, ab(2,j), ab(1,j+1), ldab-1)
 *   dpbtrs('L')  ->  dtbsv('L','N','N') then dtbsv('L','T','N')
 * in reference-BLAS loop order (no FMA). It is also the body the oracle/_ref
 * build links as dpbtrf_/dpbtrs_ (oracle/ref_driver.cpp), so oracle and
 * reference share bit-identical Poisson arithmetic. tests/test_oracle_pin.py
 * checks it against the OpenBLAS 0.3.15 copy shipped in the image (tolerance:
 * OpenBLAS kernels use FMA).
 */
#include <math.h>

#include "sk_oracle.h"

int sko_dpbtrf_lower(int n, int kd, double* ab, int ldab) {
    for (int j = 0; j < n; ++j) {
        double ajj = ab[(long)j * ldab];
        if (ajj <= 0.0) return j + 1;
        ajj = sqrt(ajj);
        ab[(long)j * ldab] = ajj;
        int kn = kd < n - 1 - j ? kd : n - 1 - j;
        if (kn > 0) {
            double r = 1.0 / ajj;
            double* x = ab + (long)j * ldab + 1;
            for (int i = 0; i < kn; ++i) x[i] = r * x[i];
            /* dsyr lower, alpha = -1: A(ii,jj) += x(ii) * (alpha * x(jj)) */
            for (int jj = 0; jj < kn; ++jj) {
                if (x[jj] != 0.0) {
                    double temp = -1.0 * x[jj];
                    double* col = ab + (long)(j + 1 + jj) * ldab;
                    for (int ii = jj; ii < kn; ++ii) col[ii - jj] = col[ii - jj] + x[ii] * temp;
                }
            }
        }
    }
    return 0;
}

void sko_dpbtrs_lower(int n, int kd, const double* ab, int ldab, double* x) {
    /* dtbsv lower, no transpose, non-unit */
    for (int j = 0; j < n; ++j) {
        if (x[j] != 0.0) {
            const double* col = ab + (long)j * ldab;
            x[j] = x[j] / col[0];
            double temp = x[j];
            int imax = n - 1 < j + kd ? n - 1 : j + kd;
            for (int i = j + 1; i <= imax; ++i) x[i] = x[i] - temp * col[i - j];
        }
    }
    /* dtbsv lower, transpose, non-unit */
    for (int j = n - 1; j >= 0; --j) {
        const double* col = ab + (long)j * ldab;
        double temp = x[j];
        int imax = n - 1 < j + kd ? n - 1 : j + kd;
        for (int i = imax; i >= j + 1; --i) temp = temp - col[i - j] * x[i];
        temp = temp / col[0];
        x[j] = temp;
    }
}
