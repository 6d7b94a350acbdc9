/* gen/genc.c -- fast C version of gen.powerlaw (identical output, verified
 * against the numpy recipe by tests/test_gen.py).  Input generation only: no
 * arithmetic of the SpMV method lives here.
 *
 * Row i: L_i = min(cap, n, floor(8.25 / sqrt(1 - u01(r(2, i))))); the diagonal
 * plus the first L_i - 1 distinct off-diagonal candidates in slot order, slot
 * s drawn from r(3, i, s) (near/far choice) and r(4, i, s) (offset/column);
 * columns sorted; values from r(5, i, position).  r(stream, a, b) is the
 * counter RNG of gen/__init__.py: splitmix64(splitmix64(key ^ a) + b * C).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t key_of(uint64_t seed, uint64_t stream) {
    return sm64(seed * 0x100000001B3ull + stream * 0x9E37ull);
}
static inline uint64_t ctr(uint64_t key, uint64_t a, uint64_t b) {
    return sm64(sm64(key ^ a) + b * 0xD1B54A32D192ED03ull);
}
static inline double u01(uint64_t bits) { return (double)(bits >> 11) * (1.0 / 9007199254740992.0); }

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* Row lengths of rows [lo, hi) into len[]; returns total nnz. */
int64_t powerlaw_lengths(int64_t n, int64_t lo, int64_t hi, uint64_t seed, int64_t cap, int64_t* len) {
    const uint64_t k2 = key_of(seed, 2);
    int64_t tot = 0;
    for (int64_t i = lo; i < hi; ++i) {
        double u = 1.0 - u01(ctr(k2, (uint64_t)i, 0));
        double L = floor(8.25 / sqrt(u));
        if (L > (double)cap) L = (double)cap;
        if (L > (double)n) L = (double)n;
        len[i - lo] = (int64_t)L;
        tot += (int64_t)L;
    }
    return tot;
}

/* Fill col/val of rows [lo, hi) given their lengths (rowptr relative, from 0). */
int powerlaw_fill(int64_t n, int64_t lo, int64_t hi, uint64_t seed, int exact, const int64_t* rowptr,
                  int32_t* col, double* val) {
    const uint64_t k3 = key_of(seed, 3), k4 = key_of(seed, 4), k5 = key_of(seed, 5);
    const int64_t w = n / 16 > 1 ? n / 16 : 1;
    int64_t cap = 0;
    for (int64_t i = lo; i < hi; ++i) {
        int64_t L = rowptr[i - lo + 1] - rowptr[i - lo];
        if (L > cap) cap = L;
    }
    /* open-addressing set of size >= 4 * cap */
    int64_t hsz = 16;
    while (hsz < 4 * cap + 16) hsz <<= 1;
    int64_t* hset = (int64_t*)malloc(sizeof(int64_t) * hsz);
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (cap + 1));
    if (!hset || !buf) return -1;
    for (int64_t i = lo; i < hi; ++i) {
        const int64_t L = rowptr[i - lo + 1] - rowptr[i - lo];
        const int64_t need = L - 1;
        int64_t hm = 16;                     /* per-row table: pow2 >= 4 L */
        while (hm < 4 * L) hm <<= 1;
        for (int64_t t = 0; t < hm; ++t) hset[t] = -1;
        int64_t have = 0;
        buf[0] = i;
        for (uint64_t s = 0; have < need; ++s) {
            const uint64_t b1 = ctr(k3, (uint64_t)i, s), b2 = ctr(k4, (uint64_t)i, s);
            const double ub = u01(b2);
            int64_t c;
            if (u01(b1) < 0.75) {
                c = i + (int64_t)floor(ub * (double)(2 * w + 1)) - w;
                if (c < 0) c = 0;
                if (c > n - 1) c = n - 1;
            } else {
                c = (int64_t)floor(ub * (double)n);
            }
            if (c == i) continue;
            int64_t h = (int64_t)((sm64((uint64_t)c) & (uint64_t)(hm - 1)));
            int dup = 0;
            while (hset[h] != -1) {
                if (hset[h] == c) { dup = 1; break; }
                h = (h + 1) & (hm - 1);
            }
            if (dup) continue;
            hset[h] = c;
            buf[1 + have++] = c;
        }
        qsort(buf, (size_t)L, sizeof(int64_t), cmp_i64);
        const int64_t base = rowptr[i - lo];
        for (int64_t p = 0; p < L; ++p) {
            col[base + p] = (int32_t)buf[p];
            const uint64_t vb = ctr(k5, (uint64_t)i, (uint64_t)p);
            if (exact) {
                int64_t t = (int64_t)(vb % 16u);
                val[base + p] = (double)(t < 8 ? t - 8 : t - 7);
            } else {
                val[base + p] = 2.0 * u01(vb) - 1.0;
            }
        }
    }
    free(hset);
    free(buf);
    return 0;
}
