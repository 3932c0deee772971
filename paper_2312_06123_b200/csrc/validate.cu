// validate.cu -- graph validation on the device for er_graph_create: the same
// checks and error classes as the host validation in abi.cu, in the same precedence:
//   column range (ER_EINVAL) / self-loop (ER_ESELFLOOP) / duplicate (ER_EDUP), first failing
//   position of each row, lowest class then lowest node over all rows;
//   symmetry (ER_EASYM, lowest node): every (v, u) has (u, v), by binary search in row u;
//   connectivity (ER_EDISCONNECTED) and non-bipartiteness (ER_EBIPARTITE): level-synchronous BFS
//   from node 0, then every arc must join levels of different parity for the graph to be bipartite.
// It needs rows sorted ascending (binary search); a graph with an unsorted row, or whose BFS needs
// more than VAL_MAX_LEVELS levels, is handed back to the host validation.

#include <string>

#include "stages.h"

namespace geer {

namespace {

constexpr int VAL_MAX_LEVELS = 1 << 14;

__device__ __forceinline__ void amin_u64(unsigned long long *p, unsigned long long v) { atomicMin(p, v); }

// Per row (one warp): first failing position's class (0 range, 1 self-loop) -> *bad as (cls << 32 | v);
// duplicates (class 2) when the row has no class-0/1 failure; unsorted rows clear *sorted.
__global__ void k_val_rows(int64_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
                           unsigned long long *__restrict__ bad, int *__restrict__ sorted, int *__restrict__ maxdeg)
{
    const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (v >= n) return;
    const int64_t e0 = off[v], e1 = off[v + 1];
    int64_t first01 = INT64_MAX;   // first position with a class-0/1 failure
    int cls01 = 0;
    bool dup = false, unsorted = false;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
        const int32_t u = cols[e];
        if ((u < 0 || u >= n || u == v) && e < first01) {
            first01 = e;
            cls01 = (u < 0 || u >= n) ? 0 : 1;
        }
        if (e > e0) {
            const int32_t p = cols[e - 1];
            if (p == u) dup = true;
            else if (p > u) unsorted = true;
        }
    }
    // warp minimum of (first01, cls)
    unsigned long long key = first01 == INT64_MAX ? ~0ull : ((unsigned long long)(first01 - e0) << 1) | (unsigned)cls01;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, key, o);
        key = t < key ? t : key;
    }
    const bool anydup = __any_sync(0xffffffffu, dup), anyuns = __any_sync(0xffffffffu, unsorted);
    if (lane == 0) {
        atomicMax(maxdeg, (int)(e1 - e0));
        if (anyuns) atomicAnd(sorted, 0);
        unsigned long long cls = ~0ull;
        if (key != ~0ull) cls = key & 1ull;
        else if (anydup && !anyuns) cls = 2;
        if (cls != ~0ull) amin_u64(bad, (cls << 32) | (unsigned long long)v);
    }
}

// Symmetry (sorted rows): every arc (v, u) has v in row u; lowest failing v -> *asym.
__global__ void k_val_sym(int64_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
                          unsigned long long *__restrict__ asym)
{
    const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (v >= n) return;
    bool miss = false;
    for (int64_t e = off[v] + lane; e < off[v + 1] && !miss; e += 32) {
        const int32_t u = cols[e];
        int64_t lo = off[u], hi = off[u + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cols[mid] < (int32_t)v) lo = mid + 1;
            else hi = mid;
        }
        if (lo >= off[u + 1] || cols[lo] != (int32_t)v) miss = true;
    }
    if (__any_sync(0xffffffffu, miss) && lane == 0) amin_u64(asym, (unsigned long long)v);
}

// One BFS level: warp per frontier node, unvisited neighbours get level L + 1 and join the next frontier.
__global__ void k_val_bfs(int64_t nf, const int32_t *__restrict__ fr, const int64_t *__restrict__ off,
                          const int32_t *__restrict__ cols, int32_t *__restrict__ level, int32_t L,
                          int32_t *__restrict__ next, unsigned long long *__restrict__ ntail)
{
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nf) return;
    const int32_t v = fr[i];
    const int64_t e1 = off[v + 1];
    for (int64_t b = off[v]; b < e1; b += 32) {
        const int64_t e = b + lane;
        bool push = false;
        int32_t u = 0;
        if (e < e1) {
            u = cols[e];
            push = level[u] == -1 && atomicCAS(&level[u], -1, L + 1) == -1;
        }
        const unsigned m = __ballot_sync(0xffffffffu, push);
        unsigned long long base = 0;
        if (lane == 0 && m) base = atomicAdd(ntail, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (push) next[base + __popc(m & ((1u << lane) - 1u))] = u;
    }
}

// Bipartite iff every arc joins levels of different parity (graph connected).
__global__ void k_val_parity(int64_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
                             const int32_t *__restrict__ level, int *__restrict__ odd)
{
    const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (v >= n) return;
    bool same = false;
    for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32)
        if (((level[v] ^ level[cols[e]]) & 1) == 0) same = true;
    if (__any_sync(0xffffffffu, same) && lane == 0) atomicOr(odd, 1);
}

}  // namespace

// Device validation of the uploaded CSR (g->d_off, g->d_cols).  Returns 1 when the host validation
// must decide (an unsorted row, or a BFS deeper than VAL_MAX_LEVELS); else 0 with *code (ER_OK or
// the first failure, *msg set), *spectral (ER_OK / ER_EDISCONNECTED / ER_EBIPARTITE), *rows_sorted
// and *max_deg filled.
int validate_device(er_graph *g, int *code, std::string *msg, int *spectral, bool *rows_sorted, int32_t *max_deg)
{
    const int64_t n = g->n;
    const cudaStream_t st = g->stream;
    unsigned long long *u64 = nullptr;
    int *i32 = nullptr;
    int32_t *level = nullptr, *fa = nullptr, *fb = nullptr;
    cudaError_t e = cudaMalloc(&u64, 3 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&i32, 4 * sizeof(int));
    if (e != cudaSuccess) return cuda_fail(e, "validate_device"), 1;
    unsigned long long hu[3] = {~0ull, ~0ull, 0ull};
    int hi[4] = {1, 0, 0, 0};   // sorted, maxdeg, odd, -
    int rc = 1;
    do {
        if (cudaMemcpy(u64, hu, sizeof(hu), cudaMemcpyHostToDevice) != cudaSuccess) break;
        if (cudaMemcpy(i32, hi, sizeof(hi), cudaMemcpyHostToDevice) != cudaSuccess) break;
        const unsigned grid = blocks_for(n * 32, 256);
        k_val_rows<<<grid, 256, 0, st>>>(n, g->d_off, g->d_cols, u64, i32, i32 + 1);
        g->launches++;
        if (cudaMemcpyAsync(hu, u64, sizeof(hu), cudaMemcpyDeviceToHost, st) != cudaSuccess) break;
        if (cudaMemcpyAsync(hi, i32, sizeof(hi), cudaMemcpyDeviceToHost, st) != cudaSuccess) break;
        if (cudaStreamSynchronize(st) != cudaSuccess) break;
        *max_deg = hi[1];
        const int cls0 = hu[0] == ~0ull ? 3 : (int)(hu[0] >> 32);
        if (cls0 <= 1 || (cls0 == 2 && hi[0])) {   // (a duplicate in an unsorted row: host precedence)
            const int cls = cls0;
            const std::string node = std::to_string(hu[0] & 0xffffffffull);
            if (cls == 0) { *code = ER_EINVAL; *msg = "col id out of range in row " + node; }
            else if (cls == 1) { *code = ER_ESELFLOOP; *msg = "self-loop at node " + node; }
            else { *code = ER_EDUP; *msg = "duplicate neighbour in row " + node; }
            rc = 0;
            break;
        }
        if (!hi[0]) break;   // unsorted rows: the host validation decides
        *rows_sorted = true;
        k_val_sym<<<grid, 256, 0, st>>>(n, g->d_off, g->d_cols, u64 + 1);
        g->launches++;
        if (cudaMemcpyAsync(hu + 1, u64 + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st) != cudaSuccess) break;
        if (cudaStreamSynchronize(st) != cudaSuccess) break;
        if (hu[1] != ~0ull) {
            *code = ER_EASYM;
            *msg = "adjacency not symmetric at node " + std::to_string(hu[1]);
            rc = 0;
            break;
        }
        // BFS from node 0
        if (cudaMalloc(&level, sizeof(int32_t) * n) != cudaSuccess) break;
        if (cudaMalloc(&fa, sizeof(int32_t) * n) != cudaSuccess) break;
        if (cudaMalloc(&fb, sizeof(int32_t) * n) != cudaSuccess) break;
        if (cudaMemsetAsync(level, 0xff, sizeof(int32_t) * n, st) != cudaSuccess) break;
        const int32_t zero = 0;
        if (cudaMemcpyAsync(level, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st) != cudaSuccess) break;
        if (cudaMemcpyAsync(fa, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st) != cudaSuccess) break;
        int64_t nf = 1, visited = 1;
        int32_t L = 0;
        bool ok = true;
        while (nf > 0 && L < VAL_MAX_LEVELS) {
            if (cudaMemsetAsync(u64 + 2, 0, sizeof(unsigned long long), st) != cudaSuccess) { ok = false; break; }
            k_val_bfs<<<blocks_for(nf * 32, 256), 256, 0, st>>>(nf, fa, g->d_off, g->d_cols, level, L, fb, u64 + 2);
            g->launches++;
            unsigned long long t = 0;
            if (cudaMemcpyAsync(&t, u64 + 2, sizeof(t), cudaMemcpyDeviceToHost, st) != cudaSuccess) { ok = false; break; }
            if (cudaStreamSynchronize(st) != cudaSuccess) { ok = false; break; }
            nf = (int64_t)t;
            visited += nf;
            std::swap(fa, fb);
            L++;
        }
        if (!ok || nf > 0) break;   // error, or a very deep BFS: host
        *spectral = ER_OK;
        if (visited != n) {
            *spectral = ER_EDISCONNECTED;
        } else {
            k_val_parity<<<grid, 256, 0, st>>>(n, g->d_off, g->d_cols, level, i32 + 2);
            g->launches++;
            int odd = 0;
            if (cudaMemcpyAsync(&odd, i32 + 2, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) break;
            if (cudaStreamSynchronize(st) != cudaSuccess) break;
            if (!odd) *spectral = ER_EBIPARTITE;
        }
        *code = ER_OK;
        rc = 0;
    } while (0);
    cudaGetLastError();
    cudaFree(u64);
    cudaFree(i32);
    if (level) cudaFree(level);
    if (fa) cudaFree(fa);
    if (fb) cudaFree(fb);
    return rc;
}

}  // namespace geer
