// rng.cuh -- counter-based Gaussian sketch generator.
//
// The reference draws N(0,1) values from one sequential mt19937_64 stream
// with Box-Muller (random.cpp:10-15; datasets.cpp:25-26).  A sequential
// stream cannot be split across 148 SMs, so Omega is generated from
// Philox4x32-10 keyed by the caller's seed with the element's linear index
// as counter: one 128-bit block per element pair -> two 64-bit draws -> the
// reference's u1, u2 -> the Box-Muller pair (cos, sin).
// oracle/idk_oracle.c:idko_omega_philox is the CPU mirror used by the tests.
#pragma once

#include <cstdint>

namespace idk {

__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c[0];
        const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c[2];
        const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n1 = static_cast<uint32_t>(p1);
        const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c[3] ^ k1;
        const uint32_t n3 = static_cast<uint32_t>(p0);
        c[0] = n0;
        c[1] = n1;
        c[2] = n2;
        c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// Elements 2j and 2j+1 share Philox block j: u1, u2 from its two 64-bit
// draws (the reference's u1 = ((x>>11)+1)*2^-53 in (0,1], u2 = (x>>11)*2^-53),
// r = sqrt(-2 ln u1), and element 2j = r cos(2 pi u2), 2j+1 = r sin(2 pi u2)
// (both Box-Muller outputs: one log, one sqrt, one sincos per two values).
__device__ __forceinline__ void philox_normal_pair(uint64_t j, uint64_t seed, double& c0, double& c1) {
    uint32_t c[4] = {static_cast<uint32_t>(j), static_cast<uint32_t>(j >> 32), 0u, 0u};
    philox4x32_10(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const uint64_t r1 = (static_cast<uint64_t>(c[1]) << 32) | c[0];
    const uint64_t r2 = (static_cast<uint64_t>(c[3]) << 32) | c[2];
    const double u1 = __dmul_rn(static_cast<double>((r1 >> 11) + 1), 0x1.0p-53);
    const double u2 = __dmul_rn(static_cast<double>(r2 >> 11), 0x1.0p-53);
    const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    double sn, cs;
    sincos(__dmul_rn(two_pi, u2), &sn, &cs);
    c0 = __dmul_rn(r, cs);
    c1 = __dmul_rn(r, sn);
}

}  // namespace idk
