// Host check of gp_rng.h against the standard library: seed_seq-seeded
// mt19937_64 words and uniform_real_distribution<double>(0, 1) draws.
#include <cstdio>
#include <random>

#include "gp_rng.h"

int main() {
    const uint64_t seeds[] = {0, 1, 2, 0xFFFFFFFFull, 0x123456789ABCDEFull, ~0ull};
    long bad = 0, n = 0;
    for (uint64_t seed : seeds)
        for (uint64_t br : {0ull, 1ull, 77ull, 4095ull, 1ull << 33, ~0ull}) {
            std::seed_seq ss{(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)br, (uint32_t)(br >> 32)};
            std::mt19937_64 ref(ss);
            std::uniform_real_distribution<double> unif(0.0, 1.0);
            uint64_t st[gp::kMtN];
            const uint32_t s[4] = {(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)br, (uint32_t)(br >> 32)};
            gp::mt64_seed(st, s);
            uint32_t pos = gp::kMtN;
            for (int i = 0; i < 1000; i++, n++) {
                if (i % 2) {
                    const double a = unif(ref), b = gp::mt64_uniform(st, &pos);
                    bad += a != b;
                } else {
                    bad += ref() != gp::mt64_next(st, &pos);
                }
            }
        }
    std::printf("draws %ld mismatches %ld\n", n, bad);
    return bad != 0;
}
