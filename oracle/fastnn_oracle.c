/*
 * fastnn_oracle.c -- plain-C restatement of the reference FastNN matching path.
 *
 * TEST INFRASTRUCTURE ONLY (see fastnn_oracle.h).  Scalar, single-threaded,
 * written for clarity; compiled with -ffp-contract=off so every fmaf() below is
 * the one rounding the reference performs and nothing else is fused.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * compiled reference (oracle/_ref/_fastnn_ref) and the reference tests' own
 * known answers (tests/test_half.cpp, tests/test_nn.cpp, tests/test_reciprocal.cpp,
 * tests/python/test_smoke.py under /root/reference/proj).
 */
#include "fastnn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ binary16 */

/* src/half.cpp:15-47.  Magnitudes >= 65520 (the first value that RNE would send
 * to infinity) and infinities clamp to 65504 and raise the flag; NaN becomes
 * the canonical quiet NaN; the sign of zero survives. */
uint16_t orc_float_to_half_bits(float x, int* saturated) {
    uint32_t u;
    memcpy(&u, &x, 4);
    const uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
    const uint32_t mag = u & 0x7FFFFFFFu;
    if (mag > 0x7F800000u) return (uint16_t)(sign | 0x7E00u);
    if (mag >= 0x477FF000u) { /* 65520.0f */
        if (saturated) *saturated = 1;
        return (uint16_t)(sign | 0x7BFFu);
    }
    if (mag == 0) return sign;
    const int e = (int)(mag >> 23) - 127; /* unbiased exponent of x */
    if (e >= -14) {                        /* lands on a normal half */
        const uint32_t frac = mag & 0x7FFFFFu;
        const uint32_t keep = frac >> 13, drop = frac & 0x1FFFu;
        uint32_t h = ((uint32_t)(e + 15) << 10) | keep;
        if (drop > 0x1000u || (drop == 0x1000u && (keep & 1u))) h += 1u; /* carry is IEEE-correct */
        return (uint16_t)(sign | h);
    }
    if (e < -25) return sign; /* below half of the smallest subnormal */
    /* subnormal half: count units of 2^-24 with round-half-even */
    const uint32_t sig = (mag & 0x7FFFFFu) | 0x800000u; /* value = sig * 2^(e-23) */
    const uint32_t sh = (uint32_t)(-(e + 1));          /* 14..24 */
    uint32_t units = sig >> sh;
    const uint32_t rem = sig & ((1u << sh) - 1u), half = 1u << (sh - 1u);
    if (rem > half || (rem == half && (units & 1u))) units += 1u;
    return (uint16_t)(sign | units); /* 0x400 is the smallest normal, as encoded */
}

/* src/half.cpp:49-64 */
float orc_half_bits_to_float(uint16_t h) {
    const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    const uint32_t ex = (h >> 10) & 0x1Fu, man = h & 0x3FFu;
    uint32_t out;
    if (ex == 0x1Fu) {
        out = sign | 0x7F800000u | (man ? ((man << 13) | 0x400000u) : 0u);
    } else if (ex == 0) {
        float v = ldexpf((float)man, -24); /* exact */
        memcpy(&out, &v, 4);
        out |= sign;
    } else {
        out = sign | ((ex + 112u) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &out, 4);
    return f;
}

float orc_to_half_round(float x, int* saturated) {
    return orc_half_bits_to_float(orc_float_to_half_bits(x, saturated));
}

static float round_counted(float v, uint64_t* count) {
    int s = 0;
    const float r = orc_to_half_round(v, &s);
    if (s && count) ++*count;
    return r;
}

/* ------------------------------------------------------------------ distance */

/* src/kernels.cpp:31-43: one fmaf per channel, in channel order; dot negated. */
float orc_pair_distance(const float* a, const float* b, uint32_t dim, int l2) {
    float acc = 0.0f;
    for (uint32_t c = 0; c < dim; ++c) {
        if (l2) {
            const float d = a[c] - b[c];
            acc = fmaf(d, d, acc);
        } else {
            acc = fmaf(a[c], b[c], acc);
        }
    }
    return l2 ? acc : -acc;
}

/* Rounds a row block to binary16 (widened back), counting saturations. */
static float* rounded_copy(const float* src, size_t n, uint64_t* count) {
    float* out = (float*)malloc(n * sizeof(float) + 1);
    for (size_t i = 0; i < n; ++i) out[i] = round_counted(src[i], count);
    return out;
}

/* Core scan with separate saturation tallies (targets / queries / distances),
 * needed to reproduce the per-backend counter law (src/nn.cpp:143-161 for the
 * single loop, src/kernels.cpp:387-398 per double-loop block). */
static void scan_split(const float* queries, uint32_t nq, const float* targets, uint32_t nt,
                       uint32_t dim, int l2, int hybrid, uint32_t* nearest, float* min_dist,
                       uint64_t* sat_t, uint64_t* sat_q, uint64_t* sat_d) {
    const float* T = targets;
    const float* Q = queries;
    float *tr = NULL, *qr = NULL;
    if (hybrid) {
        tr = rounded_copy(targets, (size_t)nt * dim, sat_t);
        qr = rounded_copy(queries, (size_t)nq * dim, sat_q);
        T = tr;
        Q = qr;
    }
    for (uint32_t q = 0; q < nq; ++q) {
        const float* qrow = Q + (size_t)q * dim;
        float best = INFINITY;
        uint32_t idx = 0;
        for (uint32_t t = 0; t < nt; ++t) {
            float d = orc_pair_distance(qrow, T + (size_t)t * dim, dim, l2);
            if (hybrid) d = round_counted(d, sat_d);
            if (d < best) { /* strict: the earliest index keeps a tie */
                best = d;
                idx = t;
            }
        }
        nearest[q] = idx;
        min_dist[q] = best;
    }
    free(tr);
    free(qr);
}

void orc_nn_scan(const float* queries, uint32_t nq, const float* targets, uint32_t nt,
                 uint32_t dim, int l2, int hybrid, uint32_t* nearest, float* min_dist,
                 uint64_t* sat) {
    uint64_t st = 0, sq = 0, sd = 0;
    scan_split(queries, nq, targets, nt, dim, l2, hybrid, nearest, min_dist, &st, &sq, &sd);
    if (sat) *sat = st + sq + sd;
}

void orc_top2(const float* queries, uint32_t nq, const float* targets, uint32_t nt, uint32_t dim,
              int l2, float* best, uint32_t* best_idx, float* second) {
    for (uint32_t q = 0; q < nq; ++q) {
        float b = INFINITY, s = INFINITY;
        uint32_t bi = 0;
        for (uint32_t t = 0; t < nt; ++t) {
            const float d = orc_pair_distance(queries + (size_t)q * dim, targets + (size_t)t * dim,
                                              dim, l2);
            if (d < b) {
                s = b;
                b = d;
                bi = t;
            } else if (d < s) {
                s = d;
            }
        }
        best[q] = b;
        best_idx[q] = bi;
        second[q] = s;
    }
}

/* ------------------------------------------------------------------ subsample */

/* src/reciprocal.cpp:12-23: n = ceil(extent/stride) cells; a single cell samples
 * the centre, otherwise stride/2 + i*stride clamped to the last index. */
static uint32_t axis_pos(uint32_t extent, uint32_t stride, uint32_t i, uint32_t n) {
    if (n == 1) return extent / 2;
    const uint32_t p = stride / 2 + i * stride;
    return p < extent ? p : extent - 1;
}

/* src/reciprocal.cpp:64-80; stride 0 derives round(sqrt(H*W/k)), at least 1. */
uint32_t orc_grid_subsample(uint32_t height, uint32_t width, uint32_t k, uint32_t stride,
                            uint32_t* out) {
    if (stride == 0) {
        if (k == 0) return 0;
        const double cells = (double)height * (double)width / (double)k;
        long s = lround(sqrt(cells));
        stride = s < 1 ? 1u : (uint32_t)s;
    }
    const uint32_t nr = (height + stride - 1) / stride, nc = (width + stride - 1) / stride;
    if (out) {
        uint32_t n = 0;
        for (uint32_t r = 0; r < nr; ++r)
            for (uint32_t c = 0; c < nc; ++c)
                out[n++] = axis_pos(height, stride, r, nr) * width + axis_pos(width, stride, c, nc);
    }
    return nr * nc;
}

/* ------------------------------------------------------------------ matcher */

static uint32_t ceil_div(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

/* One NN query of gathered rows against a whole map, with the reference's
 * per-backend fetch and saturation accounting (src/reciprocal.cpp:37-60). */
static void run_nn(const uint32_t* ids, uint32_t n, const float* qmap, const float* tmap,
                   uint32_t nt, uint32_t dim, int l2, int hybrid, uint32_t bs, int backend,
                   uint32_t* nearest, orc_report* rep) {
    float* rows = (float*)malloc((size_t)n * dim * sizeof(float) + 1);
    for (uint32_t r = 0; r < n; ++r) memcpy(rows + (size_t)r * dim, qmap + (size_t)ids[r] * dim, dim * 4);
    float* md = (float*)malloc((size_t)n * sizeof(float) + 1);
    const int hyb = backend == 3 ? 1 : (backend == 0 ? 0 : hybrid);
    uint64_t st = 0, sq = 0, sd = 0;
    scan_split(rows, n, tmap, nt, dim, l2, hyb, nearest, md, &st, &sq, &sd);
    const uint64_t nqb = ceil_div(n, bs), ntb = ceil_div(nt, bs);
    if (backend == 1) { /* double loop: B re-fetched (and re-rounded) per block pair */
        rep->a_block_fetches += nqb;
        rep->b_block_fetches += nqb * ntb;
        rep->half_saturation_events += nqb * st + ntb * sq + sd;
    } else if (backend >= 2) {
        rep->a_block_fetches += nqb;
        rep->b_block_fetches += nqb;
        rep->half_saturation_events += st + sq + sd;
    }
    free(rows);
    free(md);
}

/* src/reciprocal.cpp:97-206 */
uint32_t orc_reciprocal_match(const float* d1, uint32_t h1, uint32_t w1, const float* d2,
                              uint32_t h2, uint32_t w2, uint32_t dim, uint32_t k,
                              uint32_t stride, uint32_t max_iters, double convergence, int l2,
                              int hybrid, uint32_t block_size, int backend, uint32_t* pairs_out,
                              orc_report* rep) {
    memset(rep, 0, sizeof(*rep));
    const uint32_t p1 = h1 * w1, p2 = h2 * w2;
    const uint32_t ns = orc_grid_subsample(h1, w1, k, stride, NULL);
    uint32_t* u = (uint32_t*)malloc((size_t)ns * 4 + 4);
    uint32_t* v = (uint32_t*)malloc((size_t)ns * 4 + 4);
    uint32_t* back = (uint32_t*)malloc((size_t)ns * 4 + 4);
    unsigned char* used_i = (unsigned char*)calloc(p1 + 1, 1);
    unsigned char* used_j = (unsigned char*)calloc(p2 + 1, 1);
    orc_grid_subsample(h1, w1, k, stride, u);
    rep->samples = ns;
    uint32_t active = ns, matches = 0;
    if (active) run_nn(u, active, d1, d2, p2, dim, l2, hybrid, block_size, backend, v, rep);
    for (uint32_t t = 1; t <= max_iters && active > 0; ++t) {
        rep->iterations = t;
        run_nn(v, active, d2, d1, p1, dim, l2, hybrid, block_size, backend, back, rep);
        uint32_t kept = 0;
        for (uint32_t s = 0; s < active; ++s) {
            if (back[s] == u[s]) { /* cycle closed */
                rep->converged++;
                if (!used_i[u[s]] && !used_j[v[s]]) {
                    used_i[u[s]] = used_j[v[s]] = 1;
                    pairs_out[3 * matches + 0] = u[s];
                    pairs_out[3 * matches + 1] = v[s];
                    pairs_out[3 * matches + 2] = t;
                    matches++;
                } else {
                    rep->duplicates_dropped++;
                }
            } else { /* survivor re-enters from the back-projected pixel */
                u[kept] = back[s];
                v[kept] = v[s];
                kept++;
            }
        }
        active = kept;
        if (rep->history_len < 64) rep->active_history[rep->history_len++] = active;
        if ((double)rep->converged / (double)ns >= convergence || t == max_iters || active == 0)
            break;
        run_nn(u, active, d1, d2, p2, dim, l2, hybrid, block_size, backend, v, rep);
    }
    rep->matches_emitted = matches;
    free(u);
    free(v);
    free(back);
    free(used_i);
    free(used_j);
    return matches;
}
