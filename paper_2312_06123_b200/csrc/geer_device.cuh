// geer_device.cuh -- device helpers: Philox4x32-10, walk-checksum hash, y-table hash,
// and the closed forms of Eq. 6 / 8 / 9 / 10 written with the same operation order
// as DESIGN.md specifies (the library is compiled with -fmad=false, so no FMA
// contraction changes a rounding).
#pragma once

#include <stdint.h>

namespace geer {

// Philox4x32-10 (Salmon et al., SC'11).  Counter/key layout: DESIGN.md R10.
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        U4 n;
        n.x = hi1 ^ c.y ^ k0;
        n.y = lo1;
        n.z = hi0 ^ c.w ^ k1;
        n.w = lo0;
        c = n;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ uint64_t fmix64(uint64_t x)
{
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

// Walk checksum term (R20).
__device__ __forceinline__ uint64_t walk_hash(uint32_t q, uint32_t b, uint32_t side, uint64_t k, int32_t end)
{
    uint64_t h = fmix64((uint64_t)q + ((uint64_t)b << 32) + ((uint64_t)side << 40));
    h = fmix64(h ^ k);
    return fmix64(h ^ (uint64_t)(uint32_t)end);
}

// y-tables: buckets of YB = 4 int32 keys (one 16-byte load, the size of a rank record, so the
// walk kernel pipelines both the same way); bucket of node v in a table of 2^lgb buckets
// (multiplicative hash, top bits).
constexpr int YB = 4;
constexpr int YB_LOG = 2;
__device__ __forceinline__ uint32_t ybucket(int32_t v, int lgb)
{
    return lgb == 0 ? 0u : ((uint32_t)v * 0x9E3779B1u) >> (32 - lgb);
}

// Eq. 10.
__device__ __forceinline__ double psi_eq10(int64_t lf, double m1s, double m2s, double m1t, double m2t,
                                           double ds, double dt)
{
    const double cu = (double)((lf + 1) / 2);
    const double fl = (double)(lf / 2);
    const double a = m1s / ds + m1t / dt;
    const double b = m2s / ds + m2t / dt;
    return 2.0 * cu * a + 2.0 * fl * b;
}

__device__ __forceinline__ bool near_int(double x)
{
    const double r = rint(x);
    const double sc = fabs(x) > 1.0 ? fabs(x) : 1.0;
    return fabs(x - r) <= 1e-12 * sc;
}

}  // namespace geer
