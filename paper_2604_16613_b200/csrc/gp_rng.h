// gp_rng.h -- std::mt19937_64 seeded from a std::seed_seq of four words and
// std::uniform_real_distribution<double>(0, 1), restated bit for bit for
// host and device code (the branch generator draws its check subsets with
// them: gp_gen.cpp make_bb on the host, gp_bbgen.cuh on the device; the
// reference seeds its adaptive shots the same way, adaptive.cpp:385-387).
//
// Follows the C++ standard's definitions as libstdc++ implements them
// ([rand.util.seedseq] generate, [rand.eng.mers] seeding from a seed
// sequence, generate_canonical with 53 bits from one 64-bit draw);
// tests/test_rng.py pins it against the standard library on the host.
#pragma once
#include <stdint.h>
#if !defined(__CUDACC__) && !defined(__host__)
#define __host__
#define __device__
#endif

namespace gp {

constexpr uint32_t kMtN = 312, kMtM = 156;

// state[312] from seed_seq{s[0], s[1], s[2], s[3]} (32-bit seeds).
__host__ __device__ inline void mt64_seed(uint64_t *state, const uint32_t s[4]) {
    // seed_seq::generate into 624 32-bit words, stored in place of the state
    uint32_t *b = reinterpret_cast<uint32_t *>(state);
    const uint32_t n = 2 * kMtN, t = 11, p = (n - t) / 2, q = p + t, ns = 4, m = n;  // m = max(s + 1, n)
    for (uint32_t i = 0; i < n; i++) b[i] = 0x8b8b8b8bu;
    for (uint32_t k = 0; k < m; k++) {
        const uint32_t arg = b[k % n] ^ b[(k + p) % n] ^ b[(k + n - 1) % n];
        const uint32_t r1 = 1664525u * (arg ^ (arg >> 27));
        uint32_t r2 = r1;
        if (k == 0) r2 += ns;
        else if (k <= ns) r2 += k % n + s[k - 1];
        else r2 += k % n;
        b[(k + p) % n] += r1;
        b[(k + q) % n] += r2;
        b[k % n] = r2;
    }
    for (uint32_t k = m; k < m + n; k++) {
        const uint32_t arg = b[k % n] + b[(k + p) % n] + b[(k - 1) % n];
        const uint32_t r3 = 1566083941u * (arg ^ (arg >> 27));
        const uint32_t r4 = r3 - k % n;
        b[(k + p) % n] ^= r3;
        b[(k + q) % n] ^= r4;
        b[k % n] = r4;
    }
    // two 32-bit words per state word, low first (in place, ascending)
    bool zero = true;
    for (uint32_t i = 0; i < kMtN; i++) {
        const uint64_t lo = b[2 * i], hi = b[2 * i + 1];
        state[i] = lo | hi << 32;
        if (i == 0 ? (state[0] >> 31) != 0 : state[i] != 0) zero = false;
    }
    if (zero) state[0] = 1ull << 63;
}

__host__ __device__ inline void mt64_twist(uint64_t *x) {
    const uint64_t upper = ~0ull << 31, lower = ~upper, a = 0xB5026F5AA96619E9ull;
    for (uint32_t k = 0; k < kMtN - kMtM; k++) {
        const uint64_t y = (x[k] & upper) | (x[k + 1] & lower);
        x[k] = x[k + kMtM] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    }
    for (uint32_t k = kMtN - kMtM; k < kMtN - 1; k++) {
        const uint64_t y = (x[k] & upper) | (x[k + 1] & lower);
        x[k] = x[k + kMtM - kMtN] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    }
    const uint64_t y = (x[kMtN - 1] & upper) | (x[0] & lower);
    x[kMtN - 1] = x[kMtM - 1] ^ (y >> 1) ^ ((y & 1) ? a : 0);
}

// Next 64-bit output; *pos starts at kMtN after seeding.
__host__ __device__ inline uint64_t mt64_next(uint64_t *x, uint32_t *pos) {
    if (*pos >= kMtN) {
        mt64_twist(x);
        *pos = 0;
    }
    uint64_t z = x[(*pos)++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

// uniform_real_distribution<double>(0, 1): generate_canonical<double, 53>
// over one draw -- (double)u (round to nearest) / 2^64, kept below 1.
__host__ __device__ inline double mt64_uniform(uint64_t *x, uint32_t *pos) {
    const uint64_t u = mt64_next(x, pos);
#if defined(__CUDA_ARCH__)
    double r = __ull2double_rn(u) * 0x1p-64;
#else
    double r = (double)u * 0x1p-64;
#endif
    if (r >= 1.0) r = 0x1.fffffffffffffp-1;  // nextafter(1, 0)
    return r;
}

}  // namespace gp
