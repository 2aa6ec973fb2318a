/*
 * ccwgpu.h -- C-ABI of the B200-native CCWSIM hot path (libccwgpu.so).
 *
 * This is the drop-in boundary.  The reference (/root/reference/proj) is a
 * header-only C++20 library with no FFI layer; its public entry points for
 * the hot path are the inline functions listed beside each declaration.  A
 * maintainer binds the reference-facing C++ API to these symbols through the
 * shim in include/ccwsim_gpu.hpp; Python binds them with
 * ctypes (paper_2404_00441_b200/_abi.py).
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross the ABI.
 *  - Every function returns a ccw_status.  0 = ok; 1-7 mirror the reference
 *    exception classes (errors.hpp:9-72); >= 100 are CUDA errors.  The message
 *    (same text as the reference's exception where one exists) is available
 *    from ccw_last_error(ctx) -- or ccw_last_error(NULL) for failures that
 *    happen before a context exists.
 *  - Host buffers are caller-owned and sized from the arguments.  Device
 *    memory is owned by the context and the TI handle.
 *  - A context binds one GPU and one CUDA stream and is not thread-safe; use
 *    one context per host thread (one per GPU / rank).
 *  - All computation runs on the GPU.  There is no CPU fallback: if the
 *    device cannot be initialised every call returns CCW_ERR_CUDA.
 */
#ifndef CCWGPU_H
#define CCWGPU_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CCW_API __attribute__((visibility("default")))
#else
#define CCW_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int ccw_status;
enum {
    CCW_OK = 0,
    CCW_ERR_BOUNDS = 1,     /* ccwsim::BoundsError      (errors.hpp:15) */
    CCW_ERR_DIMENSION = 2,  /* ccwsim::DimensionError   (errors.hpp:21) */
    CCW_ERR_STRUCTURE = 3,  /* ccwsim::StructureError   (errors.hpp:27) */
    CCW_ERR_CONFIG = 4,     /* ccwsim::ConfigError      (errors.hpp:33) */
    CCW_ERR_EMPTY = 5,      /* ccwsim::EmptyInputError  (errors.hpp:38) */
    CCW_ERR_IO = 6,         /* ccwsim::IoError          (errors.hpp:50) */
    CCW_ERR_GENERIC = 7,    /* ccwsim::Error            (errors.hpp:9)  */
    CCW_ERR_DEGENERACY = 8, /* ccwsim::DegeneracyError  (errors.hpp:44) */
    CCW_ERR_CUDA = 100
};

/* OrShape (simulator.hpp:87) and Corner (simulator.hpp:95) enum orders. */
enum { CCW_OR_NONE = 0, CCW_OR_VERTICAL = 1, CCW_OR_HORIZONTAL = 2, CCW_OR_L = 3 };
enum { CCW_TOP_LEFT = 0, CCW_TOP_RIGHT = 1, CCW_BOTTOM_LEFT = 2, CCW_BOTTOM_RIGHT = 3 };

/* ccwsim::SimConfig (simulator.hpp:28-40) minus hard_data, which is passed
 * separately as (row, col, facies) int32 triples. */
typedef struct ccw_sim_config {
    int32_t sg_height;
    int32_t sg_width;
    int32_t template_size;  /* T  */
    int32_t overlap;        /* OV */
    int32_t dwt_level;      /* J  */
    int32_t candidates;     /* K  */
    int32_t n_realizations;
    int32_t scoring;        /* 0 raw, 1 normalized       (matcher.hpp:18)    */
    int32_t facies_mode;    /* 0 indicator, 1 raw_codes  (simulator.hpp:25) */
    int32_t min_cut;        /* 0 off, 1 on                                   */
    uint64_t master_seed;
    /* Literal-config extension (not in the reference; 0 = reference
     * behaviour): overlap not divisible by 2^J allowed, coarse mask = every
     * block the fine overlap touches (extract_or zeros the rest of such a
     * block), TI not divisible by 2^J used at its top-left floor(d/2^J)*2^J
     * crop.  Semantics: oracle/ccw_oracle.h. */
    int32_t any_support;
    int32_t _pad;
} ccw_sim_config;

/* ccwsim::SimDiagnostics (simulator.hpp:376-392). */
typedef struct ccw_diag {
    uint64_t seed;
    int32_t origin;
    int32_t column_major;
    int32_t work_height;
    int32_t work_width;
    int32_t placement_count;
    int32_t hard_data_count;
    int32_t pre_overwrite_mismatches;
    int32_t _pad;
    double wall_seconds;  /* host wall time of the whole batched call */
} ccw_diag;

/* ccwsim::SimTrace (simulator.hpp:395-403), flattened per realization:
 * arrays of `capacity` entries; `pasted` (capacity*T*T) may be NULL. */
typedef struct ccw_trace {
    int32_t capacity;
    int32_t count;
    int32_t* top;
    int32_t* left;
    int32_t* shape;
    int32_t* ti_row;
    int32_t* ti_col;
    uint8_t* pasted;
} ccw_trace;

/* Per-call device timing, filled when profiling is enabled on the context. */
typedef struct ccw_timing {
    double total_ms;        /* device time of the last ccw_simulate* (always filled)  */
    double ccf_ms;          /* summed device time of the CCF screen launches      */
    double select_ms;       /* summed device time of the select+paste launches    */
    int64_t ccf_launches;
    int64_t launches;       /* every kernel this library launched in the call     */
    double ccf_flop;        /* algorithmic FLOP of the CCF screen (2*ch*npos*mask) */
    double ccf_flop_ref;    /* same count with the reference's F channels          */
    int64_t waves;
    int64_t jobs;
    int64_t rescored;       /* windows rescored in fp64 (the exact-score tie groups)   */
    int64_t screened_jobs;  /* placements that went through the CCF screen            */
    int64_t ccf_variant;    /* 0 none (normalized / F=1), 1 fp32 direct, 2 tcgen05 int8, 5 fused wave kernel; 3D: 3 / 4 by block-count width (dp4a / IMAD), 6 tcgen05 int8 over the 3D im2col */
    double ccf_mma_flop;    /* tensor-core MMA FLOP issued (full Tc x Tc window, padded K) */
    int64_t groups;         /* realization groups run concurrently on separate streams */
    int64_t list_overflows; /* placements with more than 256 windows at or above the tile bound */
    double host_prep_ms;    /* host schedule build (plans + mt19937_64 draws) before launch */
    int64_t bulk_jobs;      /* placements whose tie group went to the bulk (CTA-wide) rescoring */
    int64_t shared_groups;  /* equal-score groups rescored in chunks shared across the launch's CTAs */
    int64_t d2h_bytes;      /* realization bytes copied device -> host (streamed bands are bit-packed) */
} ccw_timing;

typedef struct ccw_ctx ccw_ctx;
typedef struct ccw_ti ccw_ti;

/* ---------------------------------------------------------- context ---- */
CCW_API ccw_status ccw_ctx_create(int device, ccw_ctx** out);
CCW_API void ccw_ctx_destroy(ccw_ctx* ctx);
CCW_API const char* ccw_last_error(const ccw_ctx* ctx);
/* The cudaStream_t the context launches on (for event timing by callers). */
CCW_API void* ccw_ctx_stream(ccw_ctx* ctx);
CCW_API ccw_status ccw_ctx_set_profiling(ccw_ctx* ctx, int enabled);
CCW_API ccw_status ccw_ctx_last_timing(ccw_ctx* ctx, ccw_timing* out);
/* Selects the CCF screen kernel: 0 = auto (tcgen05 int8 when the block
 * counts fit int8, else fp32), 1 = fp32 CUDA-core direct, 2 = tcgen05 int8. */
CCW_API ccw_status ccw_ctx_set_ccf_variant(ccw_ctx* ctx, int variant);

/* Per-context options (all default to the production setting; tests use them
 * to force rarely taken paths).  Names: groups, sched_replay, norm_screen,
 * shard_fast, uniform, s16, bulk, help_min, stream_out, pack, stream_bands,
 * place_threads.  Unknown names or negative values -> CCW_ERR_CONFIG. */
CCW_API ccw_status ccw_ctx_set_option(ccw_ctx* ctx, const char* name, long long value);

/* FP32 FFMA peak of this GPU (TFLOP/s), measured with an in-library
 * microbenchmark: the roofline denominator of the CUDA-core CCF screen. */
CCW_API ccw_status ccw_measure_fp32_peak(ccw_ctx* ctx, double* tflops);
/* Integer CUDA-core peaks of the 3D screen's inner loops (TOPS, 2 ops per
 * MAC): kind 0 = IMAD (int32), kind 1 = dp4a (4 int8 MACs per lane). */
CCW_API ccw_status ccw_measure_int_peak(ccw_ctx* ctx, int kind, double* tops);
/* Dense int8 tensor-core rate (TOPS) of the CCF screen's tcgen05 MMA shape
 * (kind::i8, M=128, N=256, cta_group::1), measured with an in-library probe. */
CCW_API ccw_status ccw_measure_i8_peak(ccw_ctx* ctx, double* tops);
/* The CCF screen kernel alone (tcgen05 int8 implicit GEMM) on njobs
 * placements' weights for template_size against the TI's im2col, `iters`
 * back-to-back launches with no dependency: milliseconds per launch.  The
 * throughput the kernel reaches when it is not on the wave chain. */
CCW_API ccw_status ccw_measure_ccf_screen(ccw_ctx* ctx, ccw_ti* ti, int template_size, int njobs,
                                          int iters, double* ms_per_launch);

/* ------------------------------------------- position sharding --------- */
/* Candidate-position sharding of one simulation across ranks.
 * The reference scores every TI window of a placement on one thread
 * (ccw_score_map_channels, matcher.hpp:147-173, then top_k :177-204).  With
 * shards, the window positions 0..npos-1 (row-major, as the reference scans
 * them) are cut into S = nranks * virtual_shards contiguous ranges; shard s
 * screens and ranks only its range and produces its local top-K under the
 * reference ranking (fp64 score desc, earlier position on ties).  Per
 * placement wave the local lists are all-gathered (ncclAllGather over
 * NVLink/NVSwitch when nranks > 1) and every rank merges the S lists into
 * the global top-K -- the reference's list, because every global top-K
 * window is in its own shard's top-K -- then picks and pastes identically.
 * Every rank must make the same ccw_simulate* calls with the same arguments;
 * every rank returns the full (identical) realizations.
 *
 * nccl_id: the 128-byte ncclUniqueId from ccw_nccl_unique_id on one rank,
 * broadcast by the caller; may be NULL when nranks == 1.  virtual_shards >= 1
 * runs that many shards inside this rank, exchanged through device memory
 * (validation on one GPU).  nranks == 1 && virtual_shards == 1 switches
 * sharding off.  NCCL is loaded at run time (libnccl.so.2) on first use. */
CCW_API ccw_status ccw_nccl_unique_id(uint8_t* id128);
CCW_API ccw_status ccw_ctx_set_position_shards(ccw_ctx* ctx, int nranks, int rank,
                                               const uint8_t* nccl_id, int virtual_shards);

/* ---------------------------------------------------------- rng -------- */
/* rng.hpp:11-16 */
CCW_API uint64_t ccw_mix64(uint64_t seed, uint64_t index);

/* ------------------------------------------------------ training image - */
/* Uploads a TI (h*w codes in [0, num_facies)) and builds its level-J
 * wavelet pyramid on the device once: replaces the per-realization
 * to_indicator_planes + dwt2(...).apex of simulate_one (simulator.hpp:429-435,
 * grid.hpp:245-263, wavelet.hpp:147-171).  facies_mode as in ccw_sim_config.
 * ccw_ti_create_device takes a device pointer instead of a host pointer. */
CCW_API ccw_status ccw_ti_create(ccw_ctx* ctx, const uint8_t* cells, int h, int w, int num_facies,
                         int levels, int facies_mode, ccw_ti** out);
CCW_API ccw_status ccw_ti_create_device(ccw_ctx* ctx, const uint8_t* d_cells, int h, int w,
                                int num_facies, int levels, int facies_mode, ccw_ti** out);
CCW_API void ccw_ti_destroy(ccw_ti* ti);
/* Copies the device apex (channels x (h>>J) x (w>>J) doubles) to the host. */
CCW_API ccw_status ccw_ti_apex(ccw_ti* ti, double* out);

/* ------------------------------------------------------- simulation ---- */
/* Batched simulate_one (simulator.hpp:418-519) for n_real explicit seeds;
 * realization r of the output (n_real * sg_height * sg_width codes) is
 * bit-identical to ccwsim::simulate_one(ti, cfg, seeds[r]).  hd may be NULL.
 * diag (n_real entries) and traces (n_real entries) may be NULL.  The TI
 * handle's levels / facies_mode must match cfg. */
CCW_API ccw_status ccw_simulate(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                        const uint64_t* seeds, int n_real, const int32_t* hd, int n_hd,
                        uint8_t* out, ccw_diag* diag, ccw_trace* traces);
/* Same, writing realizations to device memory (d_out, n_real*sg cells). */
CCW_API ccw_status ccw_simulate_device(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                               const uint64_t* seeds, int n_real, const int32_t* hd, int n_hd,
                               uint8_t* d_out, ccw_diag* diag);

/* Asynchronous ccw_simulate_device, without diagnostics: returns once the
 * call is enqueued on the context's stream, so consecutive calls overlap one
 * call's host-side planning with the previous call's device work.  d_out is
 * complete, ccw_ctx_last_timing covers the call, and an error the device
 * detects is returned, after ccw_ctx_synchronize (or any later synchronous
 * call).  Page-locked seeds / hard-data arrays must stay valid until then. */
CCW_API ccw_status ccw_simulate_device_async(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                                             const uint64_t* seeds, int n_real, const int32_t* hd,
                                             int n_hd, uint8_t* d_out);
/* Wait for the context's asynchronous calls and report their errors. */
CCW_API ccw_status ccw_ctx_synchronize(ccw_ctx* ctx);
/* simulate_ensemble (simulator.hpp:523-566): seeds mix64(master, r+1), all
 * cfg->n_realizations in one batched call (the reference's `workers` knob is
 * meaningless here and is ignored by the C++ shim, which the reference's
 * worker-count-invariance contract allows). */
CCW_API ccw_status ccw_simulate_ensemble(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                                 const int32_t* hd, int n_hd, uint8_t* out, ccw_diag* diag);

/* ------------------------------------------- drop-in fp64 operators ---- */
/* dwt2_single (wavelet.hpp:69-106): in h*w -> four (h/2)*(w/2) planes. */
CCW_API ccw_status ccw_dwt2_single_f64(ccw_ctx* ctx, const double* in, int h, int w, double* a,
                               double* dh, double* dv, double* dd);
/* idwt2_single (wavelet.hpp:108-143). */
CCW_API ccw_status ccw_idwt2_single_f64(ccw_ctx* ctx, const double* a, const double* dh,
                                const double* dv, const double* dd, int hh, int hw, double* out);
/* dwt2 (wavelet.hpp:147-171).  details packed per level j=1..J as H,V,D
 * planes of (h>>j)*(w>>j) doubles; may be NULL. */
CCW_API ccw_status ccw_dwt2_f64(ccw_ctx* ctx, const double* in, int h, int w, int levels, double* apex,
                        double* details);
/* idwt2 (wavelet.hpp:174-191), same packing. */
CCW_API ccw_status ccw_idwt2_f64(ccw_ctx* ctx, const double* apex, const double* details, int h, int w,
                         int levels, double* out);
/* ccw_score_map_channels (matcher.hpp:147-173); ccw_score_map
 * (matcher.hpp:132-141) is nch = 1, scoring = 0.  ti: nch planes of
 * ti_h*ti_w; tmpl: nch planes of t_h*t_w; mask t_h*t_w in {0,1};
 * out (ti_h-t_h+1)*(ti_w-t_w+1).  Bit-identical to the reference. */
CCW_API ccw_status ccw_score_map_f64(ccw_ctx* ctx, const double* ti, const double* tmpl, int nch,
                             int ti_h, int ti_w, int t_h, int t_w, const double* mask,
                             int scoring, double* out);
/* top_k (matcher.hpp:177-204).  rows/cols/vals hold k entries; n_out gets
 * min(k, h*w). */
CCW_API ccw_status ccw_top_k_f64(ccw_ctx* ctx, const double* scores, int h, int w, int k, int32_t* rows,
                         int32_t* cols, double* vals, int* n_out);
/* select_conditional (matcher.hpp:222-241): hd = n_hd (row, col, facies)
 * template-local triples; ti = ti_h*ti_w codes. */
CCW_API ccw_status ccw_select_conditional(ccw_ctx* ctx, const int32_t* rows, const int32_t* cols,
                                  int n_cands, const int32_t* hd, int n_hd, const uint8_t* ti,
                                  int ti_h, int ti_w, int levels, int* pick, int* mismatches);
/* min_cut_stitch (simulator.hpp:328-374) on t*t patches. */
CCW_API ccw_status ccw_min_cut_stitch(ccw_ctx* ctx, const uint8_t* existing, const uint8_t* incoming,
                              int t, int shape, int vertical_on_left, int horizontal_on_top,
                              int overlap, uint8_t* out);

/* ------------------------------------- 3D extension (BASELINE c3, c4) -- */
/* The reference has no 3D.  The 3D path is the builder's
 * generalization of simulate_one (simulator.hpp:148-252,418-519) defined in
 * oracle/ccw3d_oracle.h: 3D grids (axis 2 fastest, axis 0 vertical), 8
 * corners x 6 axis orders drawn as bounded(rng, 8), bounded(rng, 6),
 * overlap = the union of the previous-side slabs, EXACT integer scores from
 * per-facies block counts, ties to the earlier row-major position, K <= 16,
 * F <= 16.  any_support = 1 is the literal-config extension (overlap not a
 * multiple of 2^J: a coarse cell is in the mask if any fine overlap cell
 * falls in its block; the TI is used at floor(d / 2^J) * 2^J). */
typedef struct ccw_sim3d_config {
    int32_t sg[3];
    int32_t template_size;
    int32_t overlap;
    int32_t dwt_level;
    int32_t candidates;
    int32_t n_realizations;
    int32_t any_support;
    int32_t _pad;
    uint64_t master_seed;
} ccw_sim3d_config;

typedef struct ccw_diag3d {
    uint64_t seed;
    int32_t corner;  /* bit a: axis a walked descending */
    int32_t order;   /* (outer, middle, inner) axis permutation index */
    int32_t work[3];
    int32_t placement_count;
    int32_t hard_data_count;
    int32_t pre_overwrite_mismatches;
    double wall_seconds;
} ccw_diag3d;

typedef struct ccw_ti3d ccw_ti3d;

/* Uploads a d0 x d1 x d2 TI (codes < num_facies <= 16) and builds its level-J
 * block counts once on the device. */
CCW_API ccw_status ccw_ti3d_create(ccw_ctx* ctx, const uint8_t* cells, int d0, int d1, int d2, int num_facies,
                                   int levels, ccw_ti3d** out);
CCW_API void ccw_ti3d_destroy(ccw_ti3d* ti);
/* validate / validate_against in 3D; ti_dims (3 ints) may be NULL.  hd holds
 * n_hd quadruples (i0, i1, i2, facies) in SG coordinates. */
CCW_API ccw_status ccw_validate_config3d(const ccw_sim3d_config* cfg, const int32_t* ti_dims, int num_facies,
                                         const int32_t* hd, int n_hd, char* msg, size_t msg_len);
/* n_real realizations with explicit seeds; out: n_real * sg0*sg1*sg2 codes
 * (host memory; _device: device memory).  diag may be NULL.  Position
 * sharding (ccw_ctx_set_position_shards) applies: shard s screens its range
 * of window boxes and the per-wave box lists are all-gathered. */
CCW_API ccw_status ccw_simulate3d(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg, const uint64_t* seeds,
                                  int n_real, const int32_t* hd, int n_hd, uint8_t* out, ccw_diag3d* diag);
CCW_API ccw_status ccw_simulate3d_device(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg,
                                         const uint64_t* seeds, int n_real, const int32_t* hd, int n_hd,
                                         uint8_t* d_out, ccw_diag3d* diag);
/* As ccw_simulate3d, plus the provenance trace (SimTrace, simulator.hpp:395-403
 * in 3D): ti_origins[(r * capacity + p) * 3 + a] = the TI fine origin pasted
 * at placement p (raster order) of realization r, for p < capacity. */
CCW_API ccw_status ccw_simulate3d_trace(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg,
                                        const uint64_t* seeds, int n_real, const int32_t* hd, int n_hd,
                                        uint8_t* out, ccw_diag3d* diag, int32_t* ti_origins, int capacity);
/* seeds mix64(master, r + 1), r < cfg->n_realizations. */
CCW_API ccw_status ccw_simulate3d_ensemble(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg,
                                           const int32_t* hd, int n_hd, uint8_t* out, ccw_diag3d* diag);

/* ------------------------------------------ validation metrics (f3) ---- */
/* metrics.hpp:68-311 on the device, over n realizations of h x w codes held
 * in device memory (on_device = 1: e.g. ccw_simulate_device's output) or in
 * host memory (copied once).  direction 0 = east_west, 1 = north_south.
 * Messages as the reference's exceptions. */
typedef struct ccw_phist ccw_phist;
/* indicator_variogram (metrics.hpp:68-112): gamma[r * max_lag + h - 1];
 * present[r] = facies occurs (may be NULL). */
CCW_API ccw_status ccw_variogram(ccw_ctx* ctx, const uint8_t* grids, int on_device, int n, int h, int w,
                                 int facies, int direction, int max_lag, double* gamma, int32_t* present);
/* connectivity_function (metrics.hpp:158-205): prob[r * max_lag + h - 1],
 * NaN where the lag has no same-facies pair (the reference's unset optional). */
CCW_API ccw_status ccw_connectivity(ccw_ctx* ctx, const uint8_t* grids, int on_device, int n, int h, int w,
                                    int facies, int direction, int max_lag, double* prob);
/* ensemble_average (metrics.hpp:208-227): out h*w doubles. */
CCW_API ccw_status ccw_ensemble_average(ccw_ctx* ctx, const uint8_t* grids, int on_device, int n, int h, int w,
                                        int facies, double* out);
/* downsample_majority (metrics.hpp:288-311): out (h/factor)*(w/factor) codes (host). */
CCW_API ccw_status ccw_downsample_majority(ccw_ctx* ctx, const uint8_t* grid, int on_device, int h, int w,
                                           int num_facies, int factor, uint8_t* out);
/* pattern_histogram (metrics.hpp:230-254), kept on the device: exact keys
 * (window^2 * ceil(log2 num_facies) <= 128 bits). */
CCW_API ccw_status ccw_pattern_histogram(ccw_ctx* ctx, const uint8_t* grid, int on_device, int h, int w,
                                         int num_facies, int window, int stride, ccw_phist** out);
CCW_API ccw_status ccw_phist_info(const ccw_phist* hist, int64_t* distinct, int64_t* total, int* window);
/* keys: distinct * window^2 codes (row-major windows), counts: distinct. */
CCW_API ccw_status ccw_phist_copy(ccw_ctx* ctx, const ccw_phist* hist, uint8_t* keys, uint64_t* counts);
CCW_API void ccw_phist_destroy(ccw_phist* hist);
/* js_divergence (metrics.hpp:258-284), base-2, clamped to [0, 1]. */
CCW_API ccw_status ccw_js_divergence(ccw_ctx* ctx, const ccw_phist* p, const ccw_phist* q, double* out);
/* anodi (metrics.hpp:318-384; the MDS step, which needs Eigen, excluded):
 * ensembles A (n_a grids) and B (n_b) of h x w codes (on_device as above),
 * the TI in host memory; per level p the grids are majority-downsampled by
 * 2^(p-1), histogrammed with `window`, and every pairwise JS divergence runs
 * on the device.  weights: levels values or NULL (uniform).  out: levels x 8
 * doubles (between_a, between_b, within_a, within_b, d_between, d_within,
 * ratio, weight). */
CCW_API ccw_status ccw_anodi(ccw_ctx* ctx, const uint8_t* grids_a, int n_a, const uint8_t* grids_b, int n_b,
                             int on_device, int h, int w, const uint8_t* ti, int ti_h, int ti_w, int num_facies,
                             int levels, int window, const double* weights, double* out, double* aggregate);

/* -------------------------------------------------- host-side helpers -- */
/* SimConfig::validate / validate_against (simulator.hpp:46-84) incl.
 * validate_hard_data (grid.hpp:151-170); ti_h/ti_w <= 0 skips the TI part. */
CCW_API ccw_status ccw_validate_config(const ccw_sim_config* cfg, int ti_h, int ti_w, int num_facies,
                               const int32_t* hd, int n_hd, char* msg, size_t msg_len);
/* plan_raster_path (simulator.hpp:148-190) given its two rng draws:
 * origin = bounded(rng, 4), column_major = (bounded(rng, 2) == 1).  The
 * caller owns the generator (the C++ shim passes its std::mt19937_64). */
CCW_API ccw_status ccw_plan_raster_path(const ccw_sim_config* cfg, int origin, int column_major,
                                int* work_h, int* work_w, int32_t* tops, int32_t* lefts,
                                int32_t* shapes, int capacity, int* count, char* msg,
                                size_t msg_len);

#ifdef __cplusplus
}
#endif

#endif /* CCWGPU_H */
