/*
 * ccw_oracle.c -- CPU restatement of the CCWSIM hot path (see ccw_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path and the "port"
 * CPU baseline.  Never linked into the product.
 *
 * Every function restates the reference algorithm in the reference's exact
 * floating-point operation order, so results are bit-identical when built
 * with -O2 -ffp-contract=off and no -march.  Reference
 * citations are /root/reference/proj/include/ccwsim/<file>:<line>.
 */
#include "ccw_oracle.h"

#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[512];

const char* ccwo_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* ------------------------------------------------------------------ rng */

/* std::mt19937_64 (the C++ standard pins its output sequence). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* rng.hpp:11-16 */
uint64_t ccwo_mix64(uint64_t seed, uint64_t index) {
    uint64_t z = seed + index * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.hpp:21-28 */
static uint64_t bounded(mt64* g, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t r = mt64_next(g);
        if (r >= threshold) return r % n;
    }
}

void ccwo_mt64_draws(uint64_t seed, uint64_t* out, int n) {
    mt64 g;
    mt64_seed(&g, seed);
    for (int i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

void ccwo_bounded_draws(uint64_t seed, const uint64_t* ns, uint64_t* out, int n) {
    mt64 g;
    mt64_seed(&g, seed);
    for (int i = 0; i < n; ++i) out[i] = bounded(&g, ns[i]);
}

/* -------------------------------------------------------------- wavelet */

static const double kS = 0.70710678118654752440084436210485; /* wavelet.hpp:17 */

/* wavelet.hpp:69-106: row pass (s*x0 + s*x1, :29-30), then column pass
 * (s*(l0 + l1), :99-102). */
int ccwo_dwt2_single(const double* in, int h, int w, double* a, double* dh, double* dv,
                     double* dd) {
    if (h % 2 != 0 || w % 2 != 0)
        return fail(CCWO_DIMENSION, "dwt2_single requires even dimensions, got %dx%d", h, w);
    const int hh = h / 2, hw = w / 2;
    double* lo = (double*)malloc(sizeof(double) * (size_t)h * hw);
    double* hi = (double*)malloc(sizeof(double) * (size_t)h * hw);
    for (int r = 0; r < h; ++r) {
        const double* x = in + (size_t)r * w;
        for (int i = 0; i < hw; ++i) {
            lo[(size_t)r * hw + i] = kS * x[2 * i] + kS * x[2 * i + 1];
            hi[(size_t)r * hw + i] = kS * x[2 * i] + (-kS) * x[2 * i + 1];
        }
    }
    for (int i = 0; i < hh; ++i) {
        const double* l0 = lo + (size_t)(2 * i) * hw;
        const double* l1 = lo + (size_t)(2 * i + 1) * hw;
        const double* h0 = hi + (size_t)(2 * i) * hw;
        const double* h1 = hi + (size_t)(2 * i + 1) * hw;
        for (int j = 0; j < hw; ++j) {
            const size_t o = (size_t)i * hw + j;
            a[o] = kS * (l0[j] + l1[j]);
            if (dh) dh[o] = kS * (l0[j] - l1[j]);
            if (dv) dv[o] = kS * (h0[j] + h1[j]);
            if (dd) dd[o] = kS * (h0[j] - h1[j]);
        }
    }
    free(lo);
    free(hi);
    return CCWO_OK;
}

/* wavelet.hpp:108-143 */
int ccwo_idwt2_single(const double* a, const double* dh, const double* dv, const double* dd,
                      int hh, int hw, double* out) {
    const int h = 2 * hh, w = 2 * hw;
    double* lo = (double*)malloc(sizeof(double) * (size_t)h * hw);
    double* hi = (double*)malloc(sizeof(double) * (size_t)h * hw);
    for (int i = 0; i < hh; ++i)
        for (int j = 0; j < hw; ++j) {
            const size_t o = (size_t)i * hw + j;
            lo[(size_t)(2 * i) * hw + j] = kS * (a[o] + dh[o]);
            lo[(size_t)(2 * i + 1) * hw + j] = kS * (a[o] - dh[o]);
            hi[(size_t)(2 * i) * hw + j] = kS * (dv[o] + dd[o]);
            hi[(size_t)(2 * i + 1) * hw + j] = kS * (dv[o] - dd[o]);
        }
    /* synthesize (wavelet.hpp:34-40): x0 = s*lo + s*hi, x1 = s*lo + (-s)*hi */
    for (int r = 0; r < h; ++r)
        for (int i = 0; i < hw; ++i) {
            const double l = lo[(size_t)r * hw + i], d = hi[(size_t)r * hw + i];
            out[(size_t)r * w + 2 * i] = kS * l + kS * d;
            out[(size_t)r * w + 2 * i + 1] = kS * l + (-kS) * d;
        }
    free(lo);
    free(hi);
    return CCWO_OK;
}

/* wavelet.hpp:147-171 */
int ccwo_dwt2(const double* in, int h, int w, int levels, double* apex, double* details) {
    if (levels < 1) return fail(CCWO_DIMENSION, "decomposition level must be >= 1");
    if (levels > 30 || h % (1 << levels) != 0 || w % (1 << levels) != 0)
        return fail(CCWO_DIMENSION, "plane %dx%d not divisible by 2^%d", h, w, levels);
    double* cur = (double*)malloc(sizeof(double) * (size_t)h * w);
    memcpy(cur, in, sizeof(double) * (size_t)h * w);
    int ch = h, cw = w;
    size_t doff = 0;
    for (int j = 1; j <= levels; ++j) {
        const int nh = ch / 2, nw = cw / 2;
        const size_t n = (size_t)nh * nw;
        double* next = (double*)malloc(sizeof(double) * n);
        double *ph = NULL, *pv = NULL, *pd = NULL;
        if (details) {
            ph = details + doff;
            pv = ph + n;
            pd = pv + n;
            doff += 3 * n;
        }
        int rc = ccwo_dwt2_single(cur, ch, cw, next, ph, pv, pd);
        free(cur);
        if (rc) {
            free(next);
            return rc;
        }
        cur = next;
        ch = nh;
        cw = nw;
    }
    memcpy(apex, cur, sizeof(double) * (size_t)ch * cw);
    free(cur);
    return CCWO_OK;
}

/* wavelet.hpp:174-191 */
int ccwo_idwt2(const double* apex, const double* details, int h, int w, int levels,
               double* out) {
    if (levels < 1) return fail(CCWO_STRUCTURE, "pyramid level count inconsistent");
    int ch = h >> levels, cw = w >> levels;
    /* offsets of each level's detail block */
    size_t offs[32];
    size_t o = 0;
    for (int j = 1; j <= levels; ++j) {
        offs[j] = o;
        o += 3 * (size_t)(h >> j) * (size_t)(w >> j);
    }
    double* cur = (double*)malloc(sizeof(double) * (size_t)ch * cw);
    memcpy(cur, apex, sizeof(double) * (size_t)ch * cw);
    for (int j = levels; j >= 1; --j) {
        const size_t n = (size_t)ch * cw;
        const double* ph = details + offs[j];
        double* next = (double*)malloc(sizeof(double) * n * 4);
        ccwo_idwt2_single(cur, ph, ph + n, ph + 2 * n, ch, cw, next);
        free(cur);
        cur = next;
        ch *= 2;
        cw *= 2;
    }
    memcpy(out, cur, sizeof(double) * (size_t)h * w);
    free(cur);
    return CCWO_OK;
}

/* -------------------------------------------------------------- matcher */

typedef struct {
    int s, t0, t1;
} run3;

/* matcher.hpp:44-61: row-major maximal runs of mask == 1. */
static int mask_runs(const double* mask, int h, int w, run3* runs) {
    int n = 0;
    for (int s = 0; s < h; ++s) {
        const double* m = mask + (size_t)s * w;
        int t = 0;
        while (t < w) {
            if (m[t] == 1.0) {
                const int t0 = t;
                while (t < w && m[t] == 1.0) ++t;
                runs[n].s = s;
                runs[n].t0 = t0;
                runs[n].t1 = t;
                ++n;
            } else {
                ++t;
            }
        }
    }
    return n;
}

/* matcher.hpp:64-81 -- the CCF, exact accumulation order. */
static void accumulate_products(const double* ti, int ti_w, const double* tmpl, int t_w,
                                const run3* runs, int nruns, double* acc, int out_h,
                                int out_w) {
    for (int x = 0; x < out_h; ++x) {
        double* out = acc + (size_t)x * out_w;
        for (int k = 0; k < nruns; ++k) {
            const int s = runs[k].s, t0 = runs[k].t0, t1 = runs[k].t1;
            const double* ti_row = ti + (size_t)(x + s) * ti_w;
            const double* tp = tmpl + (size_t)s * t_w;
            for (int y = 0; y < out_w; ++y) {
                double sum = 0.0;
                const double* a = ti_row + y + t0;
                const double* b = tp + t0;
                for (int t = t0; t < t1; ++t) sum += *a++ * *b++;
                out[y] += sum;
            }
        }
    }
}

/* matcher.hpp:84-100 */
static void accumulate_masked_squares(const double* ti, int ti_w, const run3* runs, int nruns,
                                      double* acc, int out_h, int out_w) {
    for (int x = 0; x < out_h; ++x) {
        double* out = acc + (size_t)x * out_w;
        for (int k = 0; k < nruns; ++k) {
            const int s = runs[k].s, t0 = runs[k].t0, t1 = runs[k].t1;
            const double* ti_row = ti + (size_t)(x + s) * ti_w;
            for (int y = 0; y < out_w; ++y) {
                double sum = 0.0;
                const double* a = ti_row + y + t0;
                for (int t = t0; t < t1; ++t, ++a) sum += *a * *a;
                out[y] += sum;
            }
        }
    }
}

/* matcher.hpp:102-123 */
static int check_ccw_inputs(int ti_h, int ti_w, const double* tmpl, int t_h, int t_w,
                            const double* mask) {
    if (t_h > ti_h || t_w > ti_w)
        return fail(CCWO_DIMENSION, "template %dx%d larger than TI coefficients %dx%d", t_h,
                    t_w, ti_h, ti_w);
    for (int s = 0; s < t_h; ++s)
        for (int t = 0; t < t_w; ++t) {
            const double m = mask[(size_t)s * t_w + t];
            if (m != 0.0 && m != 1.0) return fail(CCWO_STRUCTURE, "mask values must be 0 or 1");
            if (m == 0.0 && tmpl[(size_t)s * t_w + t] != 0.0)
                return fail(CCWO_STRUCTURE, "template carries nonzero values outside the mask");
        }
    return CCWO_OK;
}

#include <math.h>

/* matcher.hpp:147-173 */
int ccwo_score_map_channels(const double* ti, const double* tmpl, int nch, int ti_h, int ti_w,
                            int t_h, int t_w, const double* mask, int scoring, double* out) {
    if (nch < 1) return fail(CCWO_STRUCTURE, "channel counts disagree");
    for (int f = 0; f < nch; ++f) {
        int rc = check_ccw_inputs(ti_h, ti_w, tmpl + (size_t)f * t_h * t_w, t_h, t_w, mask);
        if (rc) return rc;
    }
    const int out_h = ti_h - t_h + 1, out_w = ti_w - t_w + 1;
    const size_t nout = (size_t)out_h * out_w;
    for (size_t i = 0; i < nout; ++i) out[i] = 0.0;
    run3* runs = (run3*)malloc(sizeof(run3) * (size_t)(t_h * t_w + 1));
    const int nruns = mask_runs(mask, t_h, t_w, runs);
    for (int f = 0; f < nch; ++f)
        accumulate_products(ti + (size_t)f * ti_h * ti_w, ti_w, tmpl + (size_t)f * t_h * t_w,
                            t_w, runs, nruns, out, out_h, out_w);
    if (scoring == 1) {
        double* nsq = (double*)calloc(nout, sizeof(double));
        for (int f = 0; f < nch; ++f)
            accumulate_masked_squares(ti + (size_t)f * ti_h * ti_w, ti_w, runs, nruns, nsq,
                                      out_h, out_w);
        for (size_t i = 0; i < nout; ++i) {
            const double n = nsq[i];
            out[i] = n > 0.0 ? out[i] / sqrt(n) : 0.0;
        }
        free(nsq);
    }
    free(runs);
    return CCWO_OK;
}

/* matcher.hpp:177-204: descending, earlier row-major location wins ties. */
int ccwo_top_k(const double* scores, int h, int w, int k, int32_t* rows, int32_t* cols,
               double* vals, int* n_out) {
    if ((size_t)h * (size_t)w == 0) return fail(CCWO_EMPTY, "top_k on empty score map");
    if (k < 1) return fail(CCWO_CONFIG, "candidate count must be >= 1");
    int n = 0;
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            const double score = scores[(size_t)r * w + c];
            if (n == k && score <= vals[n - 1]) continue;
            int pos = n;
            while (pos > 0 && vals[pos - 1] < score) --pos;
            const int last = n < k ? n : k - 1; /* entry pushed out if full */
            for (int i = last; i > pos; --i) {
                rows[i] = rows[i - 1];
                cols[i] = cols[i - 1];
                vals[i] = vals[i - 1];
            }
            rows[pos] = r;
            cols[pos] = c;
            vals[pos] = score;
            if (n < k) ++n;
        }
    *n_out = n;
    return CCWO_OK;
}

/* matcher.hpp:222-241 */
int ccwo_select_conditional(const int32_t* rows, const int32_t* cols, const double* vals,
                            int n_cands, const int32_t* hd, int n_hd, const uint8_t* ti,
                            int ti_h, int ti_w, int levels, int* pick, int* mismatches) {
    (void)vals;
    if (n_cands < 1) return fail(CCWO_EMPTY, "select_conditional on empty candidate set");
    int best = 0, best_mis = n_hd + 1;
    for (int i = 0; i < n_cands; ++i) {
        const int fr = rows[i] << levels, fc = cols[i] << levels;
        int mis = 0;
        for (int d = 0; d < n_hd; ++d) {
            const int r = fr + hd[3 * d], c = fc + hd[3 * d + 1];
            if (r < 0 || r >= ti_h || c < 0 || c >= ti_w)
                return fail(CCWO_BOUNDS, "cell (%d, %d) outside %dx%d grid", r, c, ti_h, ti_w);
            if (ti[(size_t)r * ti_w + c] != hd[3 * d + 2]) ++mis;
        }
        if (mis == 0) {
            *pick = i;
            *mismatches = 0;
            return CCWO_OK;
        }
        if (mis < best_mis) {
            best = i;
            best_mis = mis;
        }
    }
    *pick = best;
    *mismatches = best_mis;
    return CCWO_OK;
}

/* ------------------------------------------------------------ simulator */

enum { SH_NONE = 0, SH_VERT = 1, SH_HORZ = 2, SH_L = 3 };
enum { C_TL = 0, C_TR = 1, C_BL = 2, C_BR = 3 };

/* simulator.hpp:46-69 */
static int validate_cfg(const ccwo_sim_config* c) {
    if (c->sg_height < 1 || c->sg_width < 1)
        return fail(CCWO_CONFIG, "sg_size: dimensions must be positive");
    if (c->dwt_level < 1) return fail(CCWO_CONFIG, "dwt_level: must be >= 1");
    if (c->template_size < 2) return fail(CCWO_CONFIG, "template: must be >= 2");
    if (c->overlap < 1 || c->overlap >= c->template_size)
        return fail(CCWO_CONFIG, "overlap: must be in [1, template)");
    const int b = 1 << c->dwt_level;
    if (c->template_size % b != 0)
        return fail(CCWO_CONFIG, "template: %d not divisible by 2^dwt_level = %d",
                    c->template_size, b);
    if (c->overlap % b != 0 && !c->any_support)
        return fail(CCWO_CONFIG, "overlap: %d not divisible by 2^dwt_level = %d", c->overlap, b);
    if (c->candidates < 1) return fail(CCWO_CONFIG, "candidates: must be >= 1");
    if (c->n_realizations < 1) return fail(CCWO_CONFIG, "realizations: must be >= 1");
    if (c->template_size > c->sg_height || c->template_size > c->sg_width)
        return fail(CCWO_CONFIG, "template: %d exceeds simulation grid %dx%d", c->template_size,
                    c->sg_height, c->sg_width);
    return CCWO_OK;
}

/* grid.hpp:151-170 */
static int validate_hd(const int32_t* hd, int n_hd, int h, int w, int nf) {
    int* seen = NULL;
    if (n_hd > 0) {
        seen = (int*)malloc(sizeof(int) * (size_t)h * w);
        for (size_t i = 0; i < (size_t)h * w; ++i) seen[i] = -1;
    }
    for (int i = 0; i < n_hd; ++i) {
        const int r = hd[3 * i], c = hd[3 * i + 1], f = hd[3 * i + 2];
        if (r < 0 || r >= h || c < 0 || c >= w) {
            free(seen);
            return fail(CCWO_BOUNDS, "hard datum %d at (%d, %d) outside %dx%d grid", i, r, c, h, w);
        }
        if (f < 0 || f >= nf) {
            free(seen);
            return fail(CCWO_BOUNDS, "hard datum %d has facies %d outside [0, %d)", i, f, nf);
        }
        int* s = &seen[(size_t)r * w + c];
        if (*s >= 0) {
            const int prev = *s;
            free(seen);
            return fail(CCWO_STRUCTURE, "duplicate hard data at (%d, %d): entries %d and %d", r, c,
                        prev, i);
        }
        *s = i;
    }
    free(seen);
    return CCWO_OK;
}

/* simulator.hpp:72-84 */
static int validate_against(const ccwo_sim_config* c, int ti_h, int ti_w, int nf,
                            const int32_t* hd, int n_hd) {
    int rc = validate_cfg(c);
    if (rc) return rc;
    const int b = 1 << c->dwt_level;
    const int uh = c->any_support ? ti_h / b * b : ti_h, uw = c->any_support ? ti_w / b * b : ti_w;
    if (c->template_size > uh || c->template_size > uw)
        return fail(CCWO_CONFIG, "template: %d exceeds training image %dx%d", c->template_size,
                    ti_h, ti_w);
    if (!c->any_support && (ti_h % b != 0 || ti_w % b != 0))
        return fail(CCWO_CONFIG, "training image %dx%d not divisible by 2^dwt_level = %d", ti_h,
                    ti_w, b);
    if (hd) return validate_hd(hd, n_hd, c->sg_height, c->sg_width, nf);
    return CCWO_OK;
}

/* simulator.hpp:125-131 */
static int padded_extent(int sg, int t, int stride) {
    if (sg == t) return t;
    const int span = sg - t;
    const int steps = (span + stride - 1) / stride;
    return t + steps * stride;
}

typedef struct {
    int origin, column_major, work_h, work_w, count;
    int32_t *tops, *lefts, *shapes;
} plan_t;

/* simulator.hpp:148-190 */
static int make_plan(const ccwo_sim_config* cfg, mt64* rng, plan_t* p) {
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    const int t = cfg->template_size, stride = t - cfg->overlap;
    p->origin = (int)bounded(rng, 4);
    p->column_major = bounded(rng, 2) == 1;
    p->work_h = padded_extent(cfg->sg_height, t, stride);
    p->work_w = padded_extent(cfg->sg_width, t, stride);
    const int rows_asc = p->origin == C_TL || p->origin == C_TR;
    const int cols_asc = p->origin == C_TL || p->origin == C_BL;
    int nr = 0, nc = 0;
    for (int q = 0; q + t <= p->work_h; q += stride) ++nr;
    for (int q = 0; q + t <= p->work_w; q += stride) ++nc;
    int* rp = (int*)malloc(sizeof(int) * nr);
    int* cp = (int*)malloc(sizeof(int) * nc);
    for (int i = 0; i < nr; ++i) rp[i] = rows_asc ? i * stride : (nr - 1 - i) * stride;
    for (int i = 0; i < nc; ++i) cp[i] = cols_asc ? i * stride : (nc - 1 - i) * stride;
    const int* outer = p->column_major ? cp : rp;
    const int* inner = p->column_major ? rp : cp;
    const int no = p->column_major ? nc : nr, ni = p->column_major ? nr : nc;
    p->count = no * ni;
    p->tops = (int32_t*)malloc(sizeof(int32_t) * p->count);
    p->lefts = (int32_t*)malloc(sizeof(int32_t) * p->count);
    p->shapes = (int32_t*)malloc(sizeof(int32_t) * p->count);
    int k = 0;
    for (int o = 0; o < no; ++o)
        for (int i = 0; i < ni; ++i, ++k) {
            p->tops[k] = p->column_major ? inner[i] : outer[o];
            p->lefts[k] = p->column_major ? outer[o] : inner[i];
            int sh;
            if (o == 0 && i == 0)
                sh = SH_NONE;
            else if (o == 0)
                sh = p->column_major ? SH_HORZ : SH_VERT;
            else if (i == 0)
                sh = p->column_major ? SH_VERT : SH_HORZ;
            else
                sh = SH_L;
            p->shapes[k] = sh;
        }
    free(rp);
    free(cp);
    return CCWO_OK;
}

static void free_plan(plan_t* p) {
    free(p->tops);
    free(p->lefts);
    free(p->shapes);
}

int ccwo_plan_raster_path(const ccwo_sim_config* cfg, uint64_t seed, int* origin,
                          int* column_major, int* work_h, int* work_w, int32_t* tops,
                          int32_t* lefts, int32_t* shapes, int capacity, int* count) {
    mt64 g;
    mt64_seed(&g, seed);
    plan_t p;
    int rc = make_plan(cfg, &g, &p);
    if (rc) return rc;
    *origin = p.origin;
    *column_major = p.column_major;
    *work_h = p.work_h;
    *work_w = p.work_w;
    *count = p.count;
    for (int i = 0; i < p.count && i < capacity; ++i) {
        tops[i] = p.tops[i];
        lefts[i] = p.lefts[i];
        shapes[i] = p.shapes[i];
    }
    free_plan(&p);
    return CCWO_OK;
}

static int vert_on_left(int origin) { return origin == C_TL || origin == C_BL; }
static int horz_on_top(int origin) { return origin == C_TL || origin == C_TR; }

/* simulator.hpp:194-215 */
static void support_mask(int shape, int origin, int t, int ov, double* mask) {
    for (int i = 0; i < t * t; ++i) mask[i] = 0.0;
    if (shape == SH_VERT || shape == SH_L) {
        const int c0 = vert_on_left(origin) ? 0 : t - ov;
        for (int r = 0; r < t; ++r)
            for (int c = c0; c < c0 + ov; ++c) mask[r * t + c] = 1.0;
    }
    if (shape == SH_HORZ || shape == SH_L) {
        const int r0 = horz_on_top(origin) ? 0 : t - ov;
        for (int r = r0; r < r0 + ov; ++r)
            for (int c = 0; c < t; ++c) mask[r * t + c] = 1.0;
    }
}

/* simulator.hpp:286-320 */
int ccwo_min_cost_seam(const int32_t* cost, int layers, int width, int32_t* seam) {
    int* dp = (int*)malloc(sizeof(int) * (size_t)layers * width);
    int* from = (int*)malloc(sizeof(int) * (size_t)layers * width);
    for (int j = 0; j < width; ++j) {
        dp[j] = cost[j];
        from[j] = 0;
    }
    for (int l = 1; l < layers; ++l) {
        const int* prev = dp + (size_t)(l - 1) * width;
        for (int j = 0; j < width; ++j) {
            int best = prev[j], arg = j;
            if (j > 0 && prev[j - 1] < best) {
                best = prev[j - 1];
                arg = j - 1;
            }
            if (j + 1 < width && prev[j + 1] < best) {
                best = prev[j + 1];
                arg = j + 1;
            }
            if (j > 0 && prev[j - 1] == best && j - 1 < arg) arg = j - 1;
            dp[(size_t)l * width + j] = cost[(size_t)l * width + j] + best;
            from[(size_t)l * width + j] = arg;
        }
    }
    int end = 0;
    const int* last = dp + (size_t)(layers - 1) * width;
    for (int j = 1; j < width; ++j)
        if (last[j] < last[end]) end = j;
    seam[layers - 1] = end;
    for (int l = layers - 1; l > 0; --l) seam[l - 1] = from[(size_t)l * width + seam[l]];
    free(dp);
    free(from);
    return CCWO_OK;
}

/* simulator.hpp:328-374 */
int ccwo_min_cut_stitch(const uint8_t* existing, const uint8_t* incoming, int t, int shape,
                        int vertical_on_left, int horizontal_on_top, int ov, uint8_t* out) {
    memcpy(out, incoming, (size_t)t * t);
    if (shape == SH_NONE) return CCWO_OK;
    if (ov < 1 || ov >= t) return fail(CCWO_STRUCTURE, "overlap band width out of range");
    int32_t* cost = (int32_t*)malloc(sizeof(int32_t) * (size_t)t * ov);
    int32_t* seam = (int32_t*)malloc(sizeof(int32_t) * (size_t)t);
    if (shape == SH_VERT || shape == SH_L) {
        const int c0 = vertical_on_left ? 0 : t - ov;
        for (int r = 0; r < t; ++r)
            for (int j = 0; j < ov; ++j)
                cost[r * ov + j] = existing[r * t + c0 + j] != out[r * t + c0 + j] ? 1 : 0;
        ccwo_min_cost_seam(cost, t, ov, seam);
        for (int r = 0; r < t; ++r)
            for (int j = 0; j < ov; ++j) {
                const int keep = vertical_on_left ? j < seam[r] : j > seam[r];
                if (keep) out[r * t + c0 + j] = existing[r * t + c0 + j];
            }
    }
    if (shape == SH_HORZ || shape == SH_L) {
        const int r0 = horizontal_on_top ? 0 : t - ov;
        for (int c = 0; c < t; ++c)
            for (int j = 0; j < ov; ++j)
                cost[c * ov + j] = existing[(r0 + j) * t + c] != out[(r0 + j) * t + c] ? 1 : 0;
        ccwo_min_cost_seam(cost, t, ov, seam);
        for (int c = 0; c < t; ++c)
            for (int j = 0; j < ov; ++j) {
                const int keep = horizontal_on_top ? j < seam[c] : j > seam[c];
                if (keep) out[(r0 + j) * t + c] = existing[(r0 + j) * t + c];
            }
    }
    free(cost);
    free(seam);
    return CCWO_OK;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* apex of dwt2(plane, levels) (wavelet.hpp:147-171; only the apex is kept). */
static void apex_of(const double* in, int h, int w, int levels, double* apex) {
    ccwo_dwt2(in, h, w, levels, apex, NULL);
}

/* simulator.hpp:418-519 */
int ccwo_simulate_one(const uint8_t* ti, int ti_h, int ti_w, int nf, const ccwo_sim_config* cfg,
                      const int32_t* hd, int n_hd, uint64_t seed, uint8_t* out, ccwo_diag* diag,
                      ccwo_trace* trace) {
    int rc = validate_against(cfg, ti_h, ti_w, nf, hd, n_hd);
    if (rc) return rc;
    const double t_start = now_s();
    const int t = cfg->template_size, L = cfg->dwt_level, b = 1 << L, ov = cfg->overlap;
    const int nch = cfg->facies_mode == 0 ? nf : 1;
    mt64 rng;
    mt64_seed(&rng, seed);

    /* TI scoring channels at level J (simulator.hpp:429-435); with the
     * literal-config extension over the top-left uh x uw crop */
    const int hc = ti_h >> L, wc = ti_w >> L, tc = t >> L;
    const int uh = hc << L, uw = wc << L;
    const size_t tin = (size_t)uh * uw;
    double* fine = (double*)malloc(sizeof(double) * tin);
    double* ti_c = (double*)malloc(sizeof(double) * (size_t)nch * hc * wc);
    for (int f = 0; f < nch; ++f) {
        for (int r = 0; r < uh; ++r)
            for (int c = 0; c < uw; ++c) {
                const uint8_t v = ti[(size_t)r * ti_w + c];
                fine[(size_t)r * uw + c] = cfg->facies_mode == 0 ? (v == f ? 1.0 : 0.0) : (double)v;
            }
        apex_of(fine, uh, uw, L, ti_c + (size_t)f * hc * wc);
    }
    free(fine);

    plan_t plan;
    rc = make_plan(cfg, &rng, &plan);
    if (rc) {
        free(ti_c);
        return rc;
    }
    const int wh = plan.work_h, ww = plan.work_w;
    uint8_t* work = (uint8_t*)calloc((size_t)wh * ww, 1);
    uint8_t* simd = (uint8_t*)calloc((size_t)wh * ww, 1);
    const int out_h = hc - tc + 1, out_w = wc - tc + 1;
    double* orp = (double*)malloc(sizeof(double) * (size_t)nch * t * t);
    double* orc = (double*)malloc(sizeof(double) * (size_t)nch * tc * tc);
    double* fmask = (double*)malloc(sizeof(double) * (size_t)t * t);
    double* cmask = (double*)malloc(sizeof(double) * (size_t)tc * tc);
    double* scores = (double*)malloc(sizeof(double) * (size_t)out_h * out_w);
    const int K = cfg->candidates;
    int32_t* crow = (int32_t*)malloc(sizeof(int32_t) * K);
    int32_t* ccol = (int32_t*)malloc(sizeof(int32_t) * K);
    double* cval = (double*)malloc(sizeof(double) * K);
    int32_t* hdl = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(n_hd > 0 ? n_hd : 1));
    uint8_t* patch = (uint8_t*)malloc((size_t)t * t);
    uint8_t* stitched = (uint8_t*)malloc((size_t)t * t);
    uint8_t* exist = (uint8_t*)malloc((size_t)t * t);
    if (trace) trace->count = 0;

    for (int k = 0; k < plan.count && rc == CCWO_OK; ++k) {
        const int top = plan.tops[k], left = plan.lefts[k], shape = plan.shapes[k];
        int fr = 0, fc = 0;
        if (shape == SH_NONE) {
            /* simulator.hpp:450-453 */
            fr = (int)bounded(&rng, (uint64_t)((uh - t) / b + 1)) * b;
            fc = (int)bounded(&rng, (uint64_t)((uw - t) / b + 1)) * b;
        } else {
            /* extract_or (simulator.hpp:225-252) */
            support_mask(shape, plan.origin, t, ov, fmask);
            for (size_t i = 0; i < (size_t)nch * t * t; ++i) orp[i] = 0.0;
            for (int r = 0; r < t && rc == CCWO_OK; ++r)
                for (int c = 0; c < t; ++c) {
                    if (fmask[r * t + c] != 1.0) continue;
                    const size_t g = (size_t)(top + r) * ww + left + c;
                    if (!simd[g]) {
                        rc = fail(CCWO_ERROR,
                                  "internal sequencing error: overlap cell (%d, %d) not yet "
                                  "simulated",
                                  top + r, left + c);
                        break;
                    }
                    const int code = work[g];
                    if (cfg->facies_mode == 0)
                        orp[(size_t)code * t * t + r * t + c] = 1.0;
                    else
                        orp[r * t + c] = (double)code;
                }
            if (rc) break;
            for (int f = 0; f < nch; ++f)
                apex_of(orp + (size_t)f * t * t, t, t, L, orc + (size_t)f * tc * tc);
            /* coarse_mask_from_fine (simulator.hpp:256-272); the literal-config
             * extension keeps every block the overlap touches */
            for (int i = 0; i < tc; ++i)
                for (int j = 0; j < tc; ++j) {
                    const double v = fmask[(i * b) * t + j * b];
                    double any = 0.0;
                    for (int r = 0; r < b; ++r)
                        for (int c = 0; c < b; ++c) {
                            const double m = fmask[(i * b + r) * t + j * b + c];
                            if (m == 1.0) any = 1.0;
                            if (m != v && !cfg->any_support)
                                rc = fail(CCWO_ERROR,
                                          "internal error: overlap mask not block-aligned");
                        }
                    cmask[i * tc + j] = cfg->any_support ? any : v;
                }
            if (rc) break;
            rc = ccwo_score_map_channels(ti_c, orc, nch, hc, wc, tc, tc, cmask, cfg->scoring,
                                         scores);
            if (rc) break;
            int ncand = 0;
            rc = ccwo_top_k(scores, out_h, out_w, K, crow, ccol, cval, &ncand);
            if (rc) break;
            /* hd_local (simulator.hpp:467-473) */
            int nloc = 0;
            for (int d = 0; d < n_hd; ++d) {
                const int r = hd[3 * d], c = hd[3 * d + 1];
                if (r >= top && r < top + t && c >= left && c < left + t) {
                    hdl[3 * nloc] = r - top;
                    hdl[3 * nloc + 1] = c - left;
                    hdl[3 * nloc + 2] = hd[3 * d + 2];
                    ++nloc;
                }
            }
            int pick = 0;
            if (nloc > 0) {
                int mis = 0;
                rc = ccwo_select_conditional(crow, ccol, cval, ncand, hdl, nloc, ti, ti_h, ti_w, L,
                                             &pick, &mis);
                if (rc) break;
            } else {
                pick = (int)bounded(&rng, (uint64_t)ncand); /* matcher.hpp:207-211 */
            }
            fr = crow[pick] << L;
            fc = ccol[pick] << L;
        }
        /* crop + optional stitch + paste (simulator.hpp:483-493) */
        for (int r = 0; r < t; ++r) memcpy(patch + r * t, ti + (size_t)(fr + r) * ti_w + fc, t);
        const uint8_t* src = patch;
        if (cfg->min_cut && shape != SH_NONE) {
            for (int r = 0; r < t; ++r)
                memcpy(exist + r * t, work + (size_t)(top + r) * ww + left, t);
            rc = ccwo_min_cut_stitch(exist, patch, t, shape, vert_on_left(plan.origin),
                                     horz_on_top(plan.origin), ov, stitched);
            if (rc) break;
            src = stitched;
        }
        for (int r = 0; r < t; ++r) {
            memcpy(work + (size_t)(top + r) * ww + left, src + r * t, t);
            memset(simd + (size_t)(top + r) * ww + left, 1, t);
        }
        if (trace && trace->count < trace->capacity) {
            const int e = trace->count++;
            trace->top[e] = top;
            trace->left[e] = left;
            trace->shape[e] = shape;
            trace->ti_row[e] = fr;
            trace->ti_col[e] = fc;
            if (trace->pasted) memcpy(trace->pasted + (size_t)e * t * t, src, (size_t)t * t);
        }
    }

    if (rc == CCWO_OK) {
        int mism = 0;
        for (int d = 0; d < n_hd; ++d) {
            const size_t g = (size_t)hd[3 * d] * ww + hd[3 * d + 1];
            if (work[g] != hd[3 * d + 2]) ++mism;
            work[g] = (uint8_t)hd[3 * d + 2];
        }
        for (int r = 0; r < cfg->sg_height; ++r)
            memcpy(out + (size_t)r * cfg->sg_width, work + (size_t)r * ww, cfg->sg_width);
        if (diag) {
            diag->seed = seed;
            diag->origin = plan.origin;
            diag->column_major = plan.column_major;
            diag->work_height = wh;
            diag->work_width = ww;
            diag->placement_count = plan.count;
            diag->hard_data_count = n_hd;
            diag->pre_overwrite_mismatches = mism;
            diag->_pad = 0;
            diag->wall_seconds = now_s() - t_start;
        }
    }
    free(ti_c);
    free_plan(&plan);
    free(work);
    free(simd);
    free(orp);
    free(orc);
    free(fmask);
    free(cmask);
    free(scores);
    free(crow);
    free(ccol);
    free(cval);
    free(hdl);
    free(patch);
    free(stitched);
    free(exist);
    return rc;
}

/* simulator.hpp:523-566: realization r uses mix64(master, r + 1); results
 * ordered by r and independent of the worker count. */
typedef struct {
    const uint8_t* ti;
    int ti_h, ti_w, nf;
    const ccwo_sim_config* cfg;
    const int32_t* hd;
    int n_hd;
    uint8_t* out;
    ccwo_diag* diags;
    int next;
    int rc;
    char err[512];
    pthread_mutex_t mu;
} ens_t;

static void* ens_worker(void* arg) {
    ens_t* e = (ens_t*)arg;
    const size_t sg = (size_t)e->cfg->sg_height * e->cfg->sg_width;
    for (;;) {
        pthread_mutex_lock(&e->mu);
        const int r = e->rc ? e->cfg->n_realizations : e->next++;
        pthread_mutex_unlock(&e->mu);
        if (r >= e->cfg->n_realizations) return NULL;
        int rc = ccwo_simulate_one(e->ti, e->ti_h, e->ti_w, e->nf, e->cfg, e->hd, e->n_hd,
                                   ccwo_mix64(e->cfg->master_seed, (uint64_t)r + 1),
                                   e->out + (size_t)r * sg, e->diags ? &e->diags[r] : NULL, NULL);
        if (rc) {
            pthread_mutex_lock(&e->mu);
            if (!e->rc) {
                e->rc = rc;
                snprintf(e->err, sizeof e->err, "%s", g_err);
            }
            pthread_mutex_unlock(&e->mu);
            return NULL;
        }
    }
}

int ccwo_simulate_ensemble(const uint8_t* ti, int ti_h, int ti_w, int nf,
                           const ccwo_sim_config* cfg, const int32_t* hd, int n_hd, int workers,
                           uint8_t* out, ccwo_diag* diags) {
    int rc = validate_against(cfg, ti_h, ti_w, nf, hd, n_hd);
    if (rc) return rc;
    ens_t e;
    memset(&e, 0, sizeof e);
    e.ti = ti;
    e.ti_h = ti_h;
    e.ti_w = ti_w;
    e.nf = nf;
    e.cfg = cfg;
    e.hd = hd;
    e.n_hd = n_hd;
    e.out = out;
    e.diags = diags;
    pthread_mutex_init(&e.mu, NULL);
    int count = workers < 1 ? 1 : workers;
    if (count > cfg->n_realizations) count = cfg->n_realizations;
    if (count <= 1) {
        ens_worker(&e);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * count);
        for (int i = 0; i < count; ++i) pthread_create(&th[i], NULL, ens_worker, &e);
        for (int i = 0; i < count; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    pthread_mutex_destroy(&e.mu);
    if (e.rc) snprintf(g_err, sizeof g_err, "%s", e.err);
    return e.rc;
}
