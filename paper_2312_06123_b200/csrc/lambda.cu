// lambda.cu -- device Lanczos estimate of lambda = max(|lambda_2|, |lambda_n|) of P = D^-1 A
// (Eq. 6; the paper uses ARPACK for this preprocessing step).
//
// P is similar to the symmetric N = D^-1/2 A D^-1/2, whose top eigenvector u1 = sqrt(d/2m)
// (eigenvalue 1) is projected out of every vector.  Lanczos with FULL re-orthogonalisation
// (classical Gram-Schmidt applied twice against the whole stored basis, which lives on the device),
// so the extreme Ritz values converge to the extreme eigenvalues of the deflated operator without
// ghost copies.  Every LZ_CHECK steps the tridiagonal T is diagonalised on the host (implicit QL)
// and the iteration stops when the residual estimates |beta_j e_j^T y| of BOTH extreme Ritz pairs
// are below LZ_TOL.  The returned value is then
//     max( |theta_max| + ||N x_max - theta_max x_max||, |theta_min| + ||N x_min - theta_min x_min|| )
// with EXPLICIT residuals of the two extreme Ritz vectors x = Q y (unit norm), computed on the
// device: for a symmetric operator every Ritz pair (theta, x) has an eigenvalue within ||N x -
// theta x|| of theta, and the extreme Ritz values of a fully re-orthogonalised Krylov basis
// converge to the extreme eigenvalues first, so the result is an upper estimate (an underestimate
// would shorten ell and silently void Thm 3.1).  The Krylov basis is capped at LZ_BASIS_BYTES.

#include <algorithm>
#include <cmath>
#include <vector>

#include "geer_internal.h"

namespace geer {

#define CKL(call)                                           \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

static constexpr int LZ_THREADS = 256;
static constexpr int LZ_BLOCKS = 296;                       // 2 per SM
static constexpr int LZ_MAXCOLS = 512;                      // basis vectors, at most
static constexpr int LZ_CHECK = 10;                         // convergence check period
static constexpr double LZ_TOL = 1e-11;                     // residual estimate at which both ends stop
static constexpr double LZ_BASIS_BYTES = 16.0 * (1ull << 30);

__global__ void k_lz_setup(int64_t n, const int64_t *__restrict__ off, double inv2m, double *__restrict__ isd,
                           double *__restrict__ u1, double *__restrict__ q)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const double d = (double)(off[v + 1] - off[v]);
    isd[v] = 1.0 / sqrt(d);
    u1[v] = sqrt(d * inv2m);
    // deterministic pseudo-random start vector
    uint64_t x = (uint64_t)v * 0x9E3779B97F4A7C15ull + 0x1234567ull;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    q[v] = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

__global__ void k_lz_mul(int64_t n, const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ c)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) c[v] = a[v] * b[v];
}

// Partial dot products of w with the k vectors V[0..k) (row-major: V + j n) and with u1 (column k):
// part[block * (k + 1) + j].  One pass over w; the columns are swept in the block.
__global__ void __launch_bounds__(LZ_THREADS) k_lz_dots(int64_t n, int k, const double *__restrict__ V,
                                                        const double *__restrict__ u1, const double *__restrict__ w,
                                                        double *__restrict__ part)
{
    __shared__ double sh[LZ_THREADS / 32];
    for (int j = 0; j <= k; j++) {
        const double *col = j < k ? V + (size_t)j * n : u1;
        double s = 0.0;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            s += col[i] * w[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < LZ_THREADS / 32; q++) t += sh[q];
            part[(size_t)blockIdx.x * (k + 1) + j] = t;
        }
        __syncthreads();
    }
}

// c[j] = sum over blocks of part[block][j] (fixed order: deterministic).
__global__ void k_lz_dots_sum(int nblocks, int k, const double *__restrict__ part, double *__restrict__ c)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j > k) return;
    double s = 0.0;
    for (int b = 0; b < nblocks; b++) s += part[(size_t)b * (k + 1) + j];
    c[j] = s;
}

// w -= sum_j c[j] V[j] + c[k] u1 (one projection pass of classical Gram-Schmidt).
__global__ void k_lz_project(int64_t n, int k, const double *__restrict__ V, const double *__restrict__ u1,
                             const double *__restrict__ c, double *__restrict__ w)
{
    __shared__ double sc[LZ_MAXCOLS + 1];
    for (int j = threadIdx.x; j <= k; j += blockDim.x) sc[j] = c[j];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = sc[k] * u1[i];
        for (int j = 0; j < k; j++) s += sc[j] * V[(size_t)j * n + i];
        w[i] -= s;
    }
}

// x = sum_j y[j] V[j] (a Ritz vector).
__global__ void k_lz_combine(int64_t n, int k, const double *__restrict__ V, const double *__restrict__ y,
                             double *__restrict__ x)
{
    __shared__ double sy[LZ_MAXCOLS];
    for (int j = threadIdx.x; j < k; j += blockDim.x) sy[j] = y[j];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < k; j++) s += sy[j] * V[(size_t)j * n + i];
        x[i] = s;
    }
}

__global__ void k_lz_axpy(int64_t n, double a, const double *__restrict__ x, double *__restrict__ y)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] += a * x[i];
}

__global__ void k_lz_scale(int64_t n, const double *__restrict__ w, double inv, double *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = w[i] * inv;
}

// Eigen-decomposition of the symmetric tridiagonal matrix (diagonal a, off-diagonal b) by the
// implicit QL algorithm with Wilkinson shifts; eigenvalues in d (ascending after sorting), the
// eigenvectors in the columns of Z (m x m, row-major).
static bool tridiag_ql(int m, std::vector<double> a, std::vector<double> b, std::vector<double> &d,
                       std::vector<double> &Z)
{
    d = a;
    std::vector<double> e(m, 0.0);
    for (int i = 0; i + 1 < m; i++) e[i] = b[i];
    Z.assign((size_t)m * m, 0.0);
    for (int i = 0; i < m; i++) Z[(size_t)i * m + i] = 1.0;
    for (int l = 0; l < m; l++) {
        int iter = 0;
        int mm;
        do {
            for (mm = l; mm < m - 1; mm++) {
                const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
                if (std::fabs(e[mm]) <= 1e-16 * dd) break;
            }
            if (mm != l) {
                if (iter++ == 200) return false;
                double gg = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::hypot(gg, 1.0);
                gg = d[mm] - d[l] + e[l] / (gg + (gg >= 0 ? std::fabs(r) : -std::fabs(r)));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = mm - 1; i >= l; i--) {
                    double f = s * e[i];
                    const double bb = c * e[i];
                    r = std::hypot(f, gg);
                    e[i + 1] = r;
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[mm] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = gg / r;
                    gg = d[i + 1] - p;
                    r = (d[i] - gg) * s + 2.0 * c * bb;
                    p = s * r;
                    d[i + 1] = gg + p;
                    gg = c * r - bb;
                    for (int k = 0; k < m; k++) {
                        f = Z[(size_t)k * m + i + 1];
                        Z[(size_t)k * m + i + 1] = s * Z[(size_t)k * m + i] + c * f;
                        Z[(size_t)k * m + i] = c * Z[(size_t)k * m + i] - s * f;
                    }
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= p;
                e[l] = gg;
                e[mm] = 0.0;
            }
        } while (mm != l);
    }
    return true;
}

int run_estimate_lambda(er_graph *g, int iters, double *lambda_out)
{
    NvtxRange nvtx_("geer/lambda");
    const int64_t n = g->n;
    cudaStream_t st = g->stream;
    const int64_t by_mem = (int64_t)(LZ_BASIS_BYTES / (8.0 * (double)n)) - 1;
    const int m = (int)std::max<int64_t>(2, std::min<int64_t>({(int64_t)iters, n - 2, (int64_t)LZ_MAXCOLS - 1, by_mem}));
    double *V = nullptr, *buf = nullptr, *part = nullptr, *cdev = nullptr;
    CKL(cudaMalloc(&V, sizeof(double) * (size_t)n * (m + 1)));
    CKL(cudaMalloc(&buf, sizeof(double) * 5 * (size_t)n));
    CKL(cudaMalloc(&part, sizeof(double) * LZ_BLOCKS * (LZ_MAXCOLS + 1)));
    CKL(cudaMalloc(&cdev, sizeof(double) * (LZ_MAXCOLS + 1)));
    double *isd = buf, *u1 = buf + n, *w = buf + 2 * n, *ty = buf + 3 * n, *tz = buf + 4 * n;
    const unsigned B = (unsigned)((n + 255) / 256);
    std::vector<double> c(LZ_MAXCOLS + 1);
    int rc = ER_OK;
    // c[0..k] = (V[0..k), u1) . x on the host
    auto dots = [&](const double *x, int k) -> int {
        k_lz_dots<<<LZ_BLOCKS, LZ_THREADS, 0, st>>>(n, k, V, u1, x, part);
        k_lz_dots_sum<<<(k + 1 + 127) / 128, 128, 0, st>>>(LZ_BLOCKS, k, part, cdev);
        g->launches += 2;
        CKL(cudaMemcpyAsync(c.data(), cdev, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, st));
        CKL(cudaStreamSynchronize(st));
        return ER_OK;
    };
    // x <- projection of x off span(V[0..k), u1), twice (CGS2)
    auto orth = [&](double *x, int k) -> int {
        for (int pass = 0; pass < 2; pass++) {
            int r = dots(x, k);
            if (r) return r;
            k_lz_project<<<LZ_BLOCKS, LZ_THREADS, 0, st>>>(n, k, V, u1, cdev, x);
            g->launches++;
        }
        return ER_OK;
    };
    auto norm = [&](const double *x, double *out) -> int {
        k_lz_dots<<<LZ_BLOCKS, LZ_THREADS, 0, st>>>(n, 0, V, x, x, part);   // column 0 = "u1" slot = x
        k_lz_dots_sum<<<1, 128, 0, st>>>(LZ_BLOCKS, 0, part, cdev);
        g->launches += 2;
        double v = 0.0;
        CKL(cudaMemcpyAsync(&v, cdev, sizeof(double), cudaMemcpyDeviceToHost, st));
        CKL(cudaStreamSynchronize(st));
        *out = std::sqrt(v);
        return ER_OK;
    };
    // y <- N x, deflated: isd * A (isd * x) projected off u1 (by the caller's orth)
    auto apply = [&](const double *x, double *y) -> int {
        k_lz_mul<<<B, 256, 0, st>>>(n, isd, x, ty);
        g->launches++;
        int r = run_spmm(g, ty, tz, 1, 0, st);
        if (r) return r;
        k_lz_mul<<<B, 256, 0, st>>>(n, isd, tz, y);
        g->launches++;
        return ER_OK;
    };
    std::vector<double> alpha, beta, d, Z;
    int kfin = 0;
    double lam = 0.0;
    do {
        k_lz_setup<<<B, 256, 0, st>>>(n, g->d_off, 1.0 / (double)g->nnz, isd, u1, V);
        g->launches++;
        if ((rc = orth(V, 0))) break;
        double nv = 0.0;
        if ((rc = norm(V, &nv))) break;
        k_lz_scale<<<B, 256, 0, st>>>(n, V, 1.0 / nv, V);
        g->launches++;
        int k = 1;   // basis vectors V[0..k)
        for (int j = 0; j < m; j++) {
            double *qj = V + (size_t)j * n;
            if ((rc = apply(qj, w))) break;
            if ((rc = dots(w, j + 1))) break;   // c[j] = alpha_j (first projection)
            const double a = c[j];
            k_lz_project<<<LZ_BLOCKS, LZ_THREADS, 0, st>>>(n, j + 1, V, u1, cdev, w);
            g->launches++;
            if ((rc = dots(w, j + 1))) break;   // second pass (CGS2)
            k_lz_project<<<LZ_BLOCKS, LZ_THREADS, 0, st>>>(n, j + 1, V, u1, cdev, w);
            g->launches++;
            double b = 0.0;
            if ((rc = norm(w, &b))) break;
            alpha.push_back(a);
            beta.push_back(b);
            k = j + 1;
            const bool last = j + 1 == m || b < 1e-13;
            if (!last) {
                k_lz_scale<<<B, 256, 0, st>>>(n, w, 1.0 / b, V + (size_t)(j + 1) * n);
                g->launches++;
            }
            if (last || (j + 1) % LZ_CHECK == 0) {
                if (!tridiag_ql(k, alpha, beta, d, Z)) {
                    set_error(ER_ESPECTRAL, "Lanczos: tridiagonal eigensolver did not converge");
                    rc = ER_ESPECTRAL;
                    break;
                }
                int imax = 0, imin = 0;
                for (int i = 1; i < k; i++) {
                    if (d[i] > d[imax]) imax = i;
                    if (d[i] < d[imin]) imin = i;
                }
                const double emax = std::fabs(b * Z[(size_t)(k - 1) * k + imax]);
                const double emin = std::fabs(b * Z[(size_t)(k - 1) * k + imin]);
                if (last || (emax < LZ_TOL && emin < LZ_TOL)) break;
            }
        }
        if (rc) break;
        kfin = k;
        // explicit residuals of the two extreme Ritz pairs
        int imax = 0, imin = 0;
        for (int i = 1; i < kfin; i++) {
            if (d[i] > d[imax]) imax = i;
            if (d[i] < d[imin]) imin = i;
        }
        for (int side = 0; side < 2; side++) {
            const int ii = side == 0 ? imax : imin;
            std::vector<double> y(kfin);
            for (int i = 0; i < kfin; i++) y[i] = Z[(size_t)i * kfin + ii];
            CKL(cudaMemcpyAsync(cdev, y.data(), sizeof(double) * kfin, cudaMemcpyHostToDevice, st));
            k_lz_combine<<<LZ_BLOCKS, LZ_THREADS, 0, st>>>(n, kfin, V, cdev, ty);   // x (in ty)
            g->launches++;
            double nx = 0.0;
            if ((rc = norm(ty, &nx))) break;
            k_lz_scale<<<B, 256, 0, st>>>(n, ty, 1.0 / nx, ty);
            g->launches++;
            CKL(cudaMemcpyAsync(w, ty, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));   // keep x
            if ((rc = apply(w, tz))) break;   // tz = N x
            // deflate: tz -= u1 (u1 . tz)
            if ((rc = dots(tz, 0))) break;
            k_lz_project<<<LZ_BLOCKS, LZ_THREADS, 0, st>>>(n, 0, V, u1, cdev, tz);
            g->launches++;
            k_lz_axpy<<<B, 256, 0, st>>>(n, -d[ii], w, tz);   // r = N x - theta x
            g->launches++;
            double rn = 0.0;
            if ((rc = norm(tz, &rn))) break;
            lam = std::max(lam, std::fabs(d[ii]) + rn);
        }
    } while (0);
    cudaFree(V);
    cudaFree(buf);
    cudaFree(part);
    cudaFree(cdev);
    if (rc) return rc;
    if (kfin == 0) {
        set_error(ER_ESPECTRAL, "Lanczos produced no iterations");
        return ER_ESPECTRAL;
    }
    *lambda_out = std::min(lam, 1.0 - 1e-12);
    return ER_OK;
}

}  // namespace geer
