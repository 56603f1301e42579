// philox.cuh -- counter-based BIAWGN sample generator for the device channel.
//
// Replaces the reference's host channel (channel.py:36-56: PCG64 substream per
// (seed, snr_idx, frame), BPSK 1-2c, noise sigma*N(0,1), LLR 2r/sigma^2) on the hot
// path.  Philox4x32-10 (Salmon et al., SC'11) is stateless: every (frame, variable
// quad) is an independent counter, so any GPU (or any number of GPUs) can generate
// any frame range and results do not depend on how frames are sharded.
//   key     = (seed_lo, seed_hi)
//   counter = (var / 4, frame_lo, frame_hi, snr_idx | domain)
// domain 0 draws the noise, domain 1 the random word of encode mode.
#pragma once
#include <cstdint>

namespace qcl {

struct u32x4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; r++) {
        uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += W0;
        k1 += W1;
    }
    return c;
}

// (0, 1) uniform with 32 random bits, never 0 (so the log below is finite).
__device__ __forceinline__ double u01(uint32_t v) { return (v + 0.5) * 2.3283064365386963e-10; }

// Four standard normals from one Philox block (two Box-Muller pairs, FP64).
__device__ __forceinline__ void normals4(u32x4 r, double out[4]) {
    double m0 = sqrt(-2.0 * log(u01(r.x)));
    double m1 = sqrt(-2.0 * log(u01(r.z)));
    double s0, c0, s1, c1;
    sincospi(2.0 * u01(r.y), &s0, &c0);
    sincospi(2.0 * u01(r.w), &s1, &c1);
    out[0] = m0 * c0;
    out[1] = m0 * s0;
    out[2] = m1 * c1;
    out[3] = m1 * s1;
}

}  // namespace qcl
