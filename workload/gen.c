/*
 * workload/gen.c -- seeded synthetic key generator shared by the CPU oracle
 * tests and the GPU path's tests/bench.
 *
 * This module holds NONE of the sort method's arithmetic: it only produces
 * input keys.  The paper's data is "generated randomly" (§4.2);
 * the exact, integer-only, counter-based recipe is SURVEY.md §8(d):
 *
 *   mix(z)      : z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
 *                 z *= 0x94D049BB133111EB; z ^= z>>31
 *   o_seed(j)   = mix(seed + (j+1) * 0x9E3779B97F4A7C15)       (counter form)
 *   mulhi(x, R) = floor(x * R / 2^64)
 *   uniform     : key_i = mulhi(o_seed(i), R)
 *   mixture (C4): w_j = o(8i+j), j=0..7; table[t] = mulhi(o(8n+t), 1e9);
 *                 sel = mulhi(w_0, 100);
 *                 sel < 70  -> Irwin-Hall(12) normal, mean 3e8, sd 2e7, clamped
 *                 sel < 90  -> table[w_7 >> 54]
 *                 otherwise -> mulhi(w_7, 1e9)
 *
 * Every function can generate any sub-range [start, start+count) of the
 * sequence, so samples of the big configs can be regenerated cheaply.
 * Built with -fopenmp: the loops are embarrassingly parallel and the result
 * does not depend on the thread count.
 */
#include <stdint.h>

#define WL_GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t wl_mix(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

static inline uint64_t wl_out(uint64_t seed, uint64_t j) {
    return wl_mix(seed + (j + 1) * WL_GOLDEN);
}

static inline uint64_t wl_mulhi(uint64_t x, uint64_t r) {
    return (uint64_t)(((unsigned __int128)x * (unsigned __int128)r) >> 64);
}

uint64_t wl_splitmix_output(uint64_t seed, uint64_t j) { return wl_out(seed, j); }
uint64_t wl_mix64(uint64_t z) { return wl_mix(z); }

void wl_uniform_i32(int32_t *out, uint64_t seed, uint64_t range, int64_t start, int64_t count) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; i++)
        out[i] = (int32_t)wl_mulhi(wl_out(seed, (uint64_t)(start + i)), range);
}

void wl_uniform_i64(int64_t *out, uint64_t seed, uint64_t range, int64_t start, int64_t count) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; i++)
        out[i] = (int64_t)wl_mulhi(wl_out(seed, (uint64_t)(start + i)), range);
}

/* C4 mixture.  n_total fixes where the 1024-entry table is drawn from. */
void wl_mixture_table(uint64_t seed, int64_t n_total, int64_t *table1024) {
    for (int t = 0; t < 1024; t++)
        table1024[t] = (int64_t)wl_mulhi(wl_out(seed, 8ULL * (uint64_t)n_total + (uint64_t)t), 1000000000ULL);
}

void wl_mixture_i32(int32_t *out, uint64_t seed, int64_t n_total, int64_t start, int64_t count) {
    int64_t table[1024];
    wl_mixture_table(seed, n_total, table);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < count; k++) {
        uint64_t i = (uint64_t)(start + k);
        uint64_t w[8];
        for (int j = 0; j < 8; j++) w[j] = wl_out(seed, 8 * i + (uint64_t)j);
        uint64_t sel = wl_mulhi(w[0], 100);
        int64_t v;
        if (sel < 70) {
            uint64_t s = 0;
            for (int j = 1; j <= 6; j++) s += (w[j] >> 32) + (w[j] & 0xFFFFFFFFULL);
            int64_t z = (int64_t)s - (int64_t)(6ULL << 32);
            v = 300000000LL + ((z * 20000000LL) >> 32); /* arithmetic shift = floor */
            if (v < 0) v = 0;
            if (v > 999999999LL) v = 999999999LL;
        } else if (sel < 90) {
            v = table[w[7] >> 54];
        } else {
            v = (int64_t)wl_mulhi(w[7], 1000000000ULL);
        }
        out[k] = (int32_t)v;
    }
}
