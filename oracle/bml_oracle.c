/* oracle/bml_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference BML hot path, used by tests/ (and by
 * __graft_entry__.smoke()) as the CHECKER for the CUDA product path. Nothing
 * in paper_1804_07981_b200/ links, loads or calls this file.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference's own known-answer vectors (SplitMix64 seed-0 sequence, the pinned
 * N=4 seed-42 lattice, FNV-1a vectors, rule truth tables, 4-torus phase cases)
 * and against the JSON files in tests/golden/, which were produced by the UNMODIFIED
 * reference compiled from /root/reference (oracle/_ref/ref_driver, see
 * tests/golden/make_goldens.py).
 *
 * Each function cites the reference code it restates
 * (paths relative to /root/reference/proj).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EMPTY 0u
#define ORC_LR 1u
#define ORC_TB 2u

/* SplitMix64 — include/bml/seeding.hpp:11-24 (Steele/Lea/Flood constants). */
uint64_t orc_splitmix64_next(uint64_t *state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* bounded — src/seeding.cpp:11-19: reject draws >= the top multiple of m.
 * Returns 0 and sets *err = 1 for m == 0 (the reference throws). */
uint64_t orc_bounded(uint64_t *state, uint64_t m, int *err) {
    if (m == 0) {
        if (err) *err = 1;
        return 0;
    }
    const uint64_t rem = (UINT64_MAX % m + 1) % m; /* 2^64 mod m */
    const uint64_t top = 0 - rem;
    for (;;) {
        const uint64_t r = orc_splitmix64_next(state);
        if (rem == 0 || r < top) return r % m;
    }
}

/* vehicles_per_species — src/seeding.cpp:21-24: floor(rho*n*n/2) in double. */
int64_t orc_vehicles_per_species(int n, double rho) {
    return (int64_t)floor(rho * (double)n * (double)n / 2.0);
}

/* init_grid — src/seeding.cpp:26-51. Descending Fisher-Yates over the n*n
 * interior indices; first k shuffled indices become LR, next k TB. Writes the
 * dense n*n interior into `out`. Returns 0, or 1 on invalid arguments.
 * orc_init_grid_masked adds the device engine's TEST hook (include/bml_dev.h,
 * bml_dev_init_random_masked): a draw with (r & reject_mask) == 0 is rejected
 * as well, so tests can drive the rejection path the reference's own rule
 * reaches less than once per 2^32 draws. reject_mask = 0 is the reference. */
int orc_init_grid_masked(int n, double rho, uint64_t seed, uint64_t reject_mask, uint8_t *out) {
    if (n < 1 || !(rho >= 0.0 && rho <= 1.0)) return 1;
    const int64_t count = (int64_t)n * n;
    const int64_t k = orc_vehicles_per_species(n, rho);
    int64_t *cells = (int64_t *)malloc((size_t)count * sizeof(int64_t));
    if (!cells) return 2;
    for (int64_t i = 0; i < count; ++i) cells[i] = i;
    uint64_t state = seed;
    for (int64_t i = count - 1; i > 0; --i) {
        const uint64_t m = (uint64_t)(i + 1);
        const uint64_t rem = (UINT64_MAX % m + 1) % m; /* bounded(), src/seeding.cpp:11-19 */
        const uint64_t top = 0 - rem;
        uint64_t r;
        for (;;) {
            r = orc_splitmix64_next(&state);
            if ((rem == 0 || r < top) && (reject_mask == 0 || (r & reject_mask) != 0)) break;
        }
        const int64_t j = (int64_t)(r % m);
        const int64_t t = cells[i];
        cells[i] = cells[j];
        cells[j] = t;
    }
    memset(out, 0, (size_t)count);
    for (int64_t i = 0; i < 2 * k; ++i) out[cells[i]] = (uint8_t)(i < k ? ORC_LR : ORC_TB);
    free(cells);
    return 0;
}

int orc_init_grid(int n, double rho, uint64_t seed, uint8_t *out) {
    return orc_init_grid_masked(n, rho, seed, 0, out);
}

/* horizontal_rule / vertical_rule — include/bml/engine.hpp:32-42. The two
 * rules differ only in the moving species, so one function serves both. */
static inline uint8_t orc_rule(uint8_t species, uint8_t upstream, uint8_t center,
                               uint8_t downstream) {
    if (upstream == species && center == ORC_EMPTY) return species;
    if (center == species && downstream == ORC_EMPTY) return ORC_EMPTY;
    return center;
}

uint8_t orc_horizontal_rule(uint8_t l, uint8_t c, uint8_t r) { return orc_rule(ORC_LR, l, c, r); }
uint8_t orc_vertical_rule(uint8_t t, uint8_t c, uint8_t b) { return orc_rule(ORC_TB, t, c, b); }

/* naive_phase — src/engine.cpp:94-120: modulo wrap, dense n*n.
 * phase 0 = horizontal (LR), 1 = vertical (TB). */
void orc_phase(int n, const uint8_t *cur, uint8_t *next, int phase) {
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            uint8_t up, down;
            if (phase == 0) {
                up = cur[(size_t)i * n + (size_t)((j - 1 + n) % n)];
                down = cur[(size_t)i * n + (size_t)((j + 1) % n)];
            } else {
                up = cur[(size_t)((i - 1 + n) % n) * n + j];
                down = cur[(size_t)((i + 1) % n) * n + j];
            }
            next[(size_t)i * n + j] =
                orc_rule(phase == 0 ? ORC_LR : ORC_TB, up, cur[(size_t)i * n + j], down);
        }
    }
}

/* moved_in_phase — src/metrics.cpp:20-29. */
int64_t orc_moved(int n, const uint8_t *before, const uint8_t *after, int phase) {
    const uint8_t species = phase == 0 ? ORC_LR : ORC_TB;
    int64_t moved = 0;
    for (size_t i = 0; i < (size_t)n * n; ++i)
        moved += before[i] == species && after[i] == ORC_EMPTY;
    return moved;
}

/* count_vehicles — src/metrics.cpp:8-18. */
void orc_counts(int n, const uint8_t *g, int64_t *lr, int64_t *tb) {
    int64_t a = 0, b = 0;
    for (size_t i = 0; i < (size_t)n * n; ++i) {
        a += g[i] == ORC_LR;
        b += g[i] == ORC_TB;
    }
    *lr = a;
    *tb = b;
}

/* fnv1a64 — include/bml/digest.hpp:13-20; grid_digest (src/digest.cpp:5-14)
 * is this over the dense interior bytes in row-major order. */
uint64_t orc_fnv1a64(const uint8_t *p, size_t len, uint64_t h) {
    for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

uint64_t orc_digest(int n, const uint8_t *g) {
    return orc_fnv1a64(g, (size_t)n * n, 0xcbf29ce484222325ull);
}

/* step / run — src/engine.cpp:196-237: H phase then V phase per step. With
 * non-NULL metric arrays (length `steps`) the observer-path quantities are
 * recorded: moved per phase and the post-step species counts. Returns 0, or
 * 2 if allocation fails, or 3 if conservation is violated (the reference
 * throws std::logic_error, engine.cpp:219-224). */
int orc_run(int n, uint8_t *grid, int64_t steps, int64_t *lr_moved, int64_t *tb_moved,
            int64_t *lr_count, int64_t *tb_count) {
    const size_t cells = (size_t)n * n;
    uint8_t *tmp = (uint8_t *)malloc(cells);
    if (!tmp) return 2;
    int64_t lr0, tb0;
    orc_counts(n, grid, &lr0, &tb0);
    for (int64_t s = 0; s < steps; ++s) {
        orc_phase(n, grid, tmp, 0);
        if (lr_moved) lr_moved[s] = orc_moved(n, grid, tmp, 0);
        orc_phase(n, tmp, grid, 1);
        if (tb_moved) tb_moved[s] = orc_moved(n, tmp, grid, 1);
        if (lr_count || tb_count) {
            int64_t a, b;
            orc_counts(n, grid, &a, &b);
            if (lr_count) lr_count[s] = a;
            if (tb_count) tb_count[s] = b;
            if (a != lr0 || b != tb0) {
                free(tmp);
                return 3;
            }
        }
    }
    free(tmp);
    return 0;
}
