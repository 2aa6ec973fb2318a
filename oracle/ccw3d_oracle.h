/*
 * ccw3d_oracle.h -- CPU restatement of the 3D CCWSIM extension.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2404_00441_b200/,
 * include/) may link, import or call this code.  Only tests/ and bench.py's
 * cpu_baseline / --impl reference legs use it, as the checker or the CPU
 * baseline.
 *
 * The reference has no 3D.  BASELINE configs 3 and 4 are 3D,
 * so the 3D path is a builder-defined extension.  This file
 * is its NORMATIVE definition; it generalizes the reference's 2D algorithm
 * line by line:
 *
 *  - grids: uint8 codes, dims (d0, d1, d2), axis 2 fastest (row-major 3D);
 *    axis 0 is the vertical axis (wells run along it);
 *  - config (simulator.hpp:28-85): T, OV divisible by 2^J (unless
 *    any_support), T <= every SG and TI extent, TI extents divisible by 2^J
 *    (any_support: the TI is used at floor(d/2^J)*2^J -- block-aligned
 *    windows never reach the trailing cells, so no window is lost);
 *  - wavelet (wavelet.hpp:69-106): the level-J Haar apex of an indicator
 *    block is count / (2*sqrt 2)^J, so scores are computed EXACTLY from the
 *    per-facies block counts N_f (TI) and n_f (overlap); no fp64 noise, no
 *    rescoring tier (the 2D reference's ulp tie-breaking, has no
 *    3D counterpart to match);
 *  - plan (simulator.hpp:148-190): corner = bounded(rng, 8) (bit a set:
 *    axis a is walked descending), order = bounded(rng, 6) picks the
 *    (outer, middle, inner) axis permutation from kOrders; work extents and
 *    axis positions as padded_extent / axis_positions per axis;
 *  - overlap (simulator.hpp:194-252): the union of the "previous-side"
 *    slabs of width OV on every axis whose traversal index is > 0 (low side
 *    when the axis ascends, high side when it descends), full extent on the
 *    other two axes; coarse mask = blocks inside the support (any_support:
 *    blocks touching it); n_f counts only support cells;
 *  - CCF (matcher.hpp:64-81): S(p) = sum_{m in mask} sum_f N_f(p+m) n_f(m),
 *    int64, over every coarse position p of the TI (row-major order);
 *  - top_k (matcher.hpp:177-204): K largest S, ties to the earlier position;
 *  - selection (matcher.hpp:207-241, simulator.hpp:467-479): hard data in
 *    the footprint -> first candidate with no mismatch, else the fewest
 *    (earlier on ties), no draw; otherwise entries[bounded(rng, size)];
 *  - first placement (simulator.hpp:450-453): block-aligned TI origin drawn
 *    per axis, axis 0 first: bounded(rng, (ti_a - T)/B + 1) * B;
 *  - paste, hard-data overwrite + pre-overwrite mismatch count, crop
 *    (simulator.hpp:483-515); ensemble seeds mix64(master, r + 1).
 *
 * Literal-config extension (BASELINE config 4's OV 12 at J 3)
 * is the any_support flag.
 */
#ifndef CCW3D_ORACLE_H
#define CCW3D_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ccwo3_config {
    int32_t sg[3];
    int32_t template_size;
    int32_t overlap;
    int32_t dwt_level;
    int32_t candidates;
    int32_t n_realizations;
    int32_t any_support;  /* literal-config extension: any-support coarse mask, TI cropped */
    int32_t _pad;
    uint64_t master_seed;
} ccwo3_config;

typedef struct ccwo3_diag {
    uint64_t seed;
    int32_t corner;          /* bit a: axis a descending */
    int32_t order;           /* index into kOrders */
    int32_t work[3];
    int32_t placement_count;
    int32_t hard_data_count;
    int32_t pre_overwrite_mismatches;
} ccwo3_diag;

/* The (outer, middle, inner) axis permutations drawn by bounded(rng, 6). */
extern const int ccwo3_orders[6][3];

/* validate / validate_against; ti dims may be NULL (config only). */
int ccwo3_validate(const ccwo3_config* cfg, const int32_t* ti_dims, int num_facies,
                   const int32_t* hd, int n_hd);

/* Exact score map of one overlap (counts n: nf x tc^3, mask: tc^3 0/1)
 * against a TI's block counts (nf x c0 x c1 x c2); out: positions
 * (c0-tc+1)(c1-tc+1)(c2-tc+1), row-major. */
int ccwo3_score_map(const int32_t* ti_counts, const int32_t* cdims, int nf, const int32_t* or_counts,
                    const uint8_t* mask, int tc, int64_t* out);

/* Level-J block counts of a TI (nf planes of cdims = floor(d / 2^J)). */
int ccwo3_block_counts(const uint8_t* ti, const int32_t* dims, int nf, int levels, int32_t* out);

/* Plan of one seed: corner, order, work extents, placement origins (3 per
 * placement, up to capacity) and OR shapes (bit a: slab on axis a). */
int ccwo3_plan(const ccwo3_config* cfg, uint64_t seed, int* corner, int* order, int32_t* work,
               int32_t* origins, int32_t* shapes, int capacity, int* count);

/* One realization.  hd: n_hd quadruples (i0, i1, i2, facies) in SG
 * coordinates.  out: sg0*sg1*sg2 codes.  chosen (may be NULL): 3 TI fine
 * origins per placement in raster order.  threads > 1 splits every score
 * map across host threads (same result). */
int ccwo3_simulate_one(const uint8_t* ti, const int32_t* ti_dims, int num_facies,
                       const ccwo3_config* cfg, const int32_t* hd, int n_hd, uint64_t seed,
                       int threads, uint8_t* out, ccwo3_diag* diag, int32_t* chosen);

/* Realizations r = 0..n-1 with seeds mix64(master, r + 1) on `workers`
 * host threads (one realization per thread at a time). */
int ccwo3_simulate_ensemble(const uint8_t* ti, const int32_t* ti_dims, int num_facies,
                            const ccwo3_config* cfg, const int32_t* hd, int n_hd, int workers,
                            uint8_t* out, ccwo3_diag* diags);

const char* ccwo3_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
