/*
 * fastnn_oracle.h -- CPU restatement of the reference FastNN matching path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file and fastnn_oracle.c are the parity
 * checker: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load oracle/_ref/liboracle.so.  Nothing in paper_2503_10017_b200/
 * links, imports or calls it; the product runs on the GPU or raises.
 *
 * Every function restates (does not copy) the algorithm at the cited place in
 * /root/reference/proj.  The restatement is pinned against the compiled
 * reference itself (oracle/_ref/_fastnn_ref) and the reference's own known
 * answers by tests/test_oracle.py.
 */
#ifndef FASTNN_ORACLE_H
#define FASTNN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* binary16 RNE with saturation to +-65504 (flagged) -- src/half.cpp:15-47 */
uint16_t orc_float_to_half_bits(float x, int* saturated);
/* exact widening -- src/half.cpp:49-64 */
float orc_half_bits_to_float(uint16_t h);
/* round-trip -- src/half.cpp:66-72 */
float orc_to_half_round(float x, int* saturated);

/* FMA chain over channels in order; l2 != 0: sum (a-b)^2, else -(sum a*b)
 * -- src/kernels.cpp:31-43 (pair_distance_raw), :277-285 (dist_scalar) */
float orc_pair_distance(const float* a, const float* b, uint32_t dim, int l2);

/* Lowest-index strict-< nearest neighbour of every query row.
 * hybrid != 0 rounds inputs and every distance to binary16 (counted in *sat)
 * -- src/kernels.cpp:137-233 (scan_block_impl), :287-300 (tie rule),
 *    src/kernels.cpp:327-339 (target rounding), :117-125 (query rounding). */
void orc_nn_scan(const float* queries, uint32_t nq, const float* targets, uint32_t nt,
                 uint32_t dim, int l2, int hybrid, uint32_t* nearest, float* min_dist,
                 uint64_t* sat);

/* Best and second-best full-precision distance per query (parity analysis of
 * near ties; no reference counterpart -- SURVEY.md 8(a) a9). */
void orc_top2(const float* queries, uint32_t nq, const float* targets, uint32_t nt, uint32_t dim,
              int l2, float* best, uint32_t* best_idx, float* second);

/* Row-major centred grid -- src/reciprocal.cpp:12-23 (axis_positions),
 * :64-80 (grid_subsample).  Returns the count; out may be NULL to size. */
uint32_t orc_grid_subsample(uint32_t height, uint32_t width, uint32_t k, uint32_t stride,
                            uint32_t* out);

typedef struct {
    uint32_t iterations, samples, converged, matches_emitted, duplicates_dropped;
    uint64_t a_block_fetches, b_block_fetches, half_saturation_events;
    uint32_t history_len;
    uint32_t active_history[64];
} orc_report;

/* Iterative reciprocal matcher -- src/reciprocal.cpp:97-206.
 * backend: 0 bruteforce, 1 double loop, 2 single loop, 3 hybridcast.
 * pairs_out holds 3*min(samples) u32 (i, j, iteration); returns match count. */
uint32_t orc_reciprocal_match(const float* d1, uint32_t h1, uint32_t w1, const float* d2,
                              uint32_t h2, uint32_t w2, uint32_t dim, uint32_t k,
                              uint32_t stride, uint32_t max_iters, double convergence, int l2,
                              int hybrid, uint32_t block_size, int backend, uint32_t* pairs_out,
                              orc_report* report);

#ifdef __cplusplus
}
#endif
#endif
