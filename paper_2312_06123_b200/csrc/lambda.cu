// lambda.cu -- device Lanczos estimate of lambda = max(|lambda_2|, |lambda_n|) of P = D^-1 A
// (Eq. 6; the paper uses ARPACK for this preprocessing step).
//
// P is similar to the symmetric N = D^-1/2 A D^-1/2, whose top eigenvector u1 = sqrt(d/2m)
// (eigenvalue 1) is deflated explicitly every step.  Lanczos without full re-orthogonalisation;
// the extreme Ritz values of the tridiagonal T are widened by their residual bounds
// |beta_m * e_m^T y| so the returned value is an upper estimate (an underestimate would
// shorten ell and silently void Thm 3.1).  T is diagonalised on the host by cyclic Jacobi.

#include <cmath>
#include <vector>

#include "geer_internal.h"

namespace geer {

#define CKL(call)                                           \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

static constexpr int DOT_BLOCKS = 296;
static constexpr int DOT_THREADS = 256;

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

__global__ void k_lz_matvec(int64_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
                            const double *__restrict__ isd, const double *__restrict__ x, double *__restrict__ w)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    double s = 0.0;
    for (int64_t e = off[v]; e < off[v + 1]; e++) {
        const int32_t u = cols[e];
        s += isd[u] * x[u];
    }
    w[v] = isd[v] * s;
}

__global__ void k_lz_mul(int64_t n, const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ c)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) c[v] = a[v] * b[v];
}

__global__ void k_lz_dot(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                         double *__restrict__ part)
{
    __shared__ double sh[DOT_THREADS];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += a[i] * b[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = DOT_THREADS / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_lz_sum(int nparts, const double *__restrict__ part, double *__restrict__ out)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nparts; i++) s += part[i];
        *out = s;
    }
}

// w = w - a*x - b*y
__global__ void k_lz_axpy2(int64_t n, double *__restrict__ w, double a, const double *__restrict__ x, double b,
                           const double *__restrict__ y)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    w[i] = w[i] - a * x[i] - b * y[i];
}

__global__ void k_lz_scale(int64_t n, const double *__restrict__ w, double inv, double *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = w[i] * inv;
}

static void jacobi_eig(int m, std::vector<double> &A, std::vector<double> &V)
{
    V.assign((size_t)m * m, 0.0);
    for (int i = 0; i < m; i++) V[(size_t)i * m + i] = 1.0;
    for (int sweep = 0; sweep < 100; sweep++) {
        double off = 0.0, diag = 0.0;
        for (int p = 0; p < m; p++) {
            diag += A[(size_t)p * m + p] * A[(size_t)p * m + p];
            for (int q = p + 1; q < m; q++) off += A[(size_t)p * m + q] * A[(size_t)p * m + q];
        }
        if (off <= 1e-32 * (diag + 1e-300)) break;
        for (int p = 0; p < m; p++) {
            for (int q = p + 1; q < m; q++) {
                const double apq = A[(size_t)p * m + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double app = A[(size_t)p * m + p], aqq = A[(size_t)q * m + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < m; k++) {
                    const double akp = A[(size_t)k * m + p], akq = A[(size_t)k * m + q];
                    A[(size_t)k * m + p] = c * akp - s * akq;
                    A[(size_t)k * m + q] = s * akp + c * akq;
                }
                for (int k = 0; k < m; k++) {
                    const double apk = A[(size_t)p * m + k], aqk = A[(size_t)q * m + k];
                    A[(size_t)p * m + k] = c * apk - s * aqk;
                    A[(size_t)q * m + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < m; k++) {
                    const double vkp = V[(size_t)k * m + p], vkq = V[(size_t)k * m + q];
                    V[(size_t)k * m + p] = c * vkp - s * vkq;
                    V[(size_t)k * m + q] = s * vkp + c * vkq;
                }
            }
        }
    }
}

int run_estimate_lambda(er_graph *g, int iters, double *lambda_out)
{
    const int64_t n = g->n;
    cudaStream_t st = g->stream;
    const int m = (int)std::min<int64_t>(iters, std::min<int64_t>(n - 1, 400));
    double *buf = nullptr, *part = nullptr, *scal = nullptr;
    CKL(cudaMalloc(&buf, sizeof(double) * 7 * n));
    CKL(cudaMalloc(&part, sizeof(double) * DOT_BLOCKS));
    CKL(cudaMalloc(&scal, sizeof(double) * 4));
    double *isd = buf, *u1 = buf + n, *qp = buf + 2 * n, *q = buf + 3 * n, *w = buf + 4 * n, *ty = buf + 5 * n,
           *tz = buf + 6 * n;
    const unsigned B = (unsigned)((n + 255) / 256);
    int rc = ER_OK;
    auto dot = [&](const double *a, const double *b, double *out) -> int {
        k_lz_dot<<<DOT_BLOCKS, DOT_THREADS, 0, st>>>(n, a, b, part);
        k_lz_sum<<<1, 32, 0, st>>>(DOT_BLOCKS, part, scal);
        g->launches += 2;
        CKL(cudaMemcpyAsync(out, scal, sizeof(double), cudaMemcpyDeviceToHost, st));
        CKL(cudaStreamSynchronize(st));
        return ER_OK;
    };
    std::vector<double> alpha, beta;
    do {
        k_lz_setup<<<B, 256, 0, st>>>(n, g->d_off, 1.0 / (double)g->nnz, isd, u1, q);
        g->launches++;
        CKL(cudaMemsetAsync(qp, 0, sizeof(double) * n, st));
        double d = 0.0;
        if ((rc = dot(u1, q, &d))) break;
        k_lz_axpy2<<<B, 256, 0, st>>>(n, q, d, u1, 0.0, u1);
        g->launches++;
        if ((rc = dot(q, q, &d))) break;
        k_lz_scale<<<B, 256, 0, st>>>(n, q, 1.0 / std::sqrt(d), q);
        g->launches++;
        double bprev = 0.0;
        for (int j = 0; j < m; j++) {
            // w = N q = D^-1/2 A D^-1/2 q, the A product on K9 (load-balanced over hub rows)
            k_lz_mul<<<B, 256, 0, st>>>(n, isd, q, ty);
            g->launches++;
            if ((rc = run_spmm(g, ty, tz, 1, 0, st))) break;
            k_lz_mul<<<B, 256, 0, st>>>(n, isd, tz, w);
            g->launches++;
            double a = 0.0;
            if ((rc = dot(q, w, &a))) break;
            k_lz_axpy2<<<B, 256, 0, st>>>(n, w, a, q, bprev, qp);
            g->launches++;
            double du = 0.0;
            if ((rc = dot(u1, w, &du))) break;
            k_lz_axpy2<<<B, 256, 0, st>>>(n, w, du, u1, 0.0, u1);
            g->launches++;
            double bb = 0.0;
            if ((rc = dot(w, w, &bb))) break;
            const double b = std::sqrt(bb);
            alpha.push_back(a);
            beta.push_back(b);
            if (b < 1e-14) break;
            std::swap(qp, q);  // qp <- q
            k_lz_scale<<<B, 256, 0, st>>>(n, w, 1.0 / b, q);
            g->launches++;
            bprev = b;
        }
    } while (0);
    cudaFree(buf);
    cudaFree(part);
    cudaFree(scal);
    if (rc) return rc;
    const int mm = (int)alpha.size();
    if (mm == 0) {
        set_error(ER_ESPECTRAL, "Lanczos produced no iterations");
        return ER_ESPECTRAL;
    }
    std::vector<double> T((size_t)mm * mm, 0.0), V;
    for (int i = 0; i < mm; i++) {
        T[(size_t)i * mm + i] = alpha[i];
        if (i + 1 < mm) T[(size_t)i * mm + i + 1] = T[(size_t)(i + 1) * mm + i] = beta[i];
    }
    jacobi_eig(mm, T, V);
    // extreme Ritz values of the deflated operator, widened by their residual bounds
    const double blast = beta[mm - 1];
    int jmax = 0, jmin = 0;
    for (int j = 1; j < mm; j++) {
        if (T[(size_t)j * mm + j] > T[(size_t)jmax * mm + jmax]) jmax = j;
        if (T[(size_t)j * mm + j] < T[(size_t)jmin * mm + jmin]) jmin = j;
    }
    const double rmax = std::fabs(blast * V[(size_t)(mm - 1) * mm + jmax]);
    const double rmin = std::fabs(blast * V[(size_t)(mm - 1) * mm + jmin]);
    const double lam = std::max(std::fabs(T[(size_t)jmax * mm + jmax]) + rmax,
                                std::fabs(T[(size_t)jmin * mm + jmin]) + rmin);
    *lambda_out = std::min(lam, 1.0 - 1e-12);
    return ER_OK;
}

}  // namespace geer
