/*
 * ccw3d_oracle.c -- CPU restatement of the 3D CCWSIM extension (normative
 * definition in ccw3d_oracle.h).  TEST INFRASTRUCTURE ONLY.
 *
 * Each step cites the 2D reference code it generalizes
 * (/root/reference/proj/include/ccwsim/*.hpp).
 */
#define _POSIX_C_SOURCE 200809L
#include "ccw3d_oracle.h"

#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* ccwo3_last_error(void) { return g_err; }

enum { E_BOUNDS = 1, E_DIMENSION = 2, E_STRUCTURE = 3, E_CONFIG = 4, E_EMPTY = 5, E_ERROR = 7 };

const int ccwo3_orders[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

/* ---------------------------------------------------------------- rng ---- */
/* std::mt19937_64 (sequence fixed by the C++ standard) and rng.hpp:11-28. */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt_seed(mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static uint64_t bounded(mt64* g, uint64_t n) { /* rng.hpp:21-28 */
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t r = mt_next(g);
        if (r >= threshold) return r % n;
    }
}

static uint64_t mix64(uint64_t seed, uint64_t index) { /* rng.hpp:11-16 */
    uint64_t z = seed + index * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------ config ----- */
static int validate_cfg(const ccwo3_config* c) { /* simulator.hpp:46-69 */
    if (c->sg[0] < 1 || c->sg[1] < 1 || c->sg[2] < 1)
        return fail(E_CONFIG, "sg_size: dimensions must be positive");
    if (c->dwt_level < 1) return fail(E_CONFIG, "dwt_level: must be >= 1");
    if (c->dwt_level > 10) return fail(E_CONFIG, "dwt_level: must be <= 10");
    if (c->template_size < 2) return fail(E_CONFIG, "template: must be >= 2");
    if (c->overlap < 1 || c->overlap >= c->template_size)
        return fail(E_CONFIG, "overlap: must be in [1, template)");
    const int b = 1 << c->dwt_level;
    if (c->template_size % b != 0)
        return fail(E_CONFIG, "template: %d not divisible by 2^dwt_level = %d", c->template_size, b);
    if (!c->any_support && c->overlap % b != 0)
        return fail(E_CONFIG, "overlap: %d not divisible by 2^dwt_level = %d", c->overlap, b);
    if (c->candidates < 1) return fail(E_CONFIG, "candidates: must be >= 1");
    if (c->n_realizations < 1) return fail(E_CONFIG, "realizations: must be >= 1");
    for (int a = 0; a < 3; ++a)
        if (c->template_size > c->sg[a])
            return fail(E_CONFIG, "template: %d exceeds simulation grid %dx%dx%d", c->template_size,
                        c->sg[0], c->sg[1], c->sg[2]);
    return 0;
}

int ccwo3_validate(const ccwo3_config* c, const int32_t* ti, int nf, const int32_t* hd, int n_hd) {
    int e = validate_cfg(c);
    if (e) return e;
    if (!ti) return 0;
    const int b = 1 << c->dwt_level;
    if (ti[0] < 1 || ti[1] < 1 || ti[2] < 1) return fail(E_DIMENSION, "grid dimensions must be positive");
    if (nf < 1 || nf > 255) return fail(E_DIMENSION, "num_facies must be in [1, 255]");
    for (int a = 0; a < 3; ++a) {
        const int used = c->any_support ? ti[a] / b * b : ti[a];
        if (c->template_size > used)
            return fail(E_CONFIG, "template: %d exceeds training image %dx%dx%d", c->template_size, ti[0],
                        ti[1], ti[2]);
    }
    if (!c->any_support && (ti[0] % b || ti[1] % b || ti[2] % b))
        return fail(E_CONFIG, "training image %dx%dx%d not divisible by 2^dwt_level = %d", ti[0], ti[1], ti[2], b);
    /* grid.hpp:151-170, in 3D */
    const size_t n = (size_t)c->sg[0] * c->sg[1] * c->sg[2];
    uint8_t* seen = n_hd > 0 ? calloc(n, 1) : NULL;
    for (int i = 0; i < n_hd; ++i) {
        const int* d = hd + 4 * i;
        if (d[0] < 0 || d[0] >= c->sg[0] || d[1] < 0 || d[1] >= c->sg[1] || d[2] < 0 || d[2] >= c->sg[2]) {
            free(seen);
            return fail(E_BOUNDS, "hard datum %d at (%d, %d, %d) outside %dx%dx%d grid", i, d[0], d[1], d[2],
                        c->sg[0], c->sg[1], c->sg[2]);
        }
        if (d[3] < 0 || d[3] >= nf) {
            free(seen);
            return fail(E_BOUNDS, "hard datum %d has facies %d outside [0, %d)", i, d[3], nf);
        }
        const size_t cell = ((size_t)d[0] * c->sg[1] + d[1]) * c->sg[2] + d[2];
        if (seen[cell]) {
            free(seen);
            return fail(E_STRUCTURE, "duplicate hard data at (%d, %d, %d)", d[0], d[1], d[2]);
        }
        seen[cell] = 1;
    }
    free(seen);
    return 0;
}

/* --------------------------------------------------------- wavelet ------- */
int ccwo3_block_counts(const uint8_t* ti, const int32_t* dims, int nf, int levels, int32_t* out) {
    const int b = 1 << levels;
    const int c0 = dims[0] / b, c1 = dims[1] / b, c2 = dims[2] / b;
    const size_t nc = (size_t)c0 * c1 * c2;
    memset(out, 0, sizeof(int32_t) * nc * nf);
    for (int i0 = 0; i0 < c0 * b; ++i0)
        for (int i1 = 0; i1 < c1 * b; ++i1)
            for (int i2 = 0; i2 < c2 * b; ++i2) {
                const int f = ti[((size_t)i0 * dims[1] + i1) * dims[2] + i2];
                if (f < 0 || f >= nf) return fail(E_BOUNDS, "cell holds code %d outside [0, %d)", f, nf);
                out[(size_t)f * nc + ((size_t)(i0 / b) * c1 + i1 / b) * c2 + i2 / b] += 1;
            }
    return 0;
}

/* ------------------------------------------------------------ CCF -------- */
typedef struct {
    const int32_t* ti; /* nf x c0 x c1 x c2 counts */
    int c[3], nf, tc;
    int nm;            /* mask cells */
    const long* moff;  /* offset of mask cell m in a counts plane */
    const int32_t* w;  /* nm x nf overlap counts */
    int o[3];
    int64_t* out;
    int p_lo, p_hi;    /* range of the first position axis */
} score_job;

static void* score_rows(void* arg) { /* matcher.hpp:64-81 */
    const score_job* s = (const score_job*)arg;
    const size_t plane = (size_t)s->c[0] * s->c[1] * s->c[2];
    for (int p0 = s->p_lo; p0 < s->p_hi; ++p0)
        for (int p1 = 0; p1 < s->o[1]; ++p1)
            for (int p2 = 0; p2 < s->o[2]; ++p2) {
                const long base = ((long)p0 * s->c[1] + p1) * s->c[2] + p2;
                int64_t acc = 0;
                for (int m = 0; m < s->nm; ++m) {
                    const int32_t* wm = s->w + (size_t)m * s->nf;
                    const long q = base + s->moff[m];
                    for (int f = 0; f < s->nf; ++f)
                        if (wm[f]) acc += (int64_t)s->ti[(size_t)f * plane + q] * wm[f];
                }
                s->out[((size_t)p0 * s->o[1] + p1) * s->o[2] + p2] = acc;
            }
    return NULL;
}

static void score_map(const int32_t* ti, const int* c, int nf, int tc, const int32_t* n /* nf x tc^3 */,
                      const uint8_t* mask, int threads, int64_t* out) {
    int o[3] = {c[0] - tc + 1, c[1] - tc + 1, c[2] - tc + 1};
    const int nt3 = tc * tc * tc;
    long* moff = malloc(sizeof(long) * nt3);
    int32_t* w = malloc(sizeof(int32_t) * (size_t)nt3 * nf);
    int nm = 0;
    for (int m0 = 0; m0 < tc; ++m0)  /* mask cells in row-major order (matcher.hpp:44-61) */
        for (int m1 = 0; m1 < tc; ++m1)
            for (int m2 = 0; m2 < tc; ++m2) {
                const int m = (m0 * tc + m1) * tc + m2;
                if (!mask[m]) continue;
                moff[nm] = ((long)m0 * c[1] + m1) * c[2] + m2;
                for (int f = 0; f < nf; ++f) w[(size_t)nm * nf + f] = n[(size_t)f * nt3 + m];
                ++nm;
            }
    if (threads < 1) threads = 1;
    if (threads > o[0]) threads = o[0];
    score_job* jobs = malloc(sizeof(score_job) * threads);
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) {
        score_job* s = &jobs[t];
        s->ti = ti;
        memcpy(s->c, c, sizeof s->c);
        memcpy(s->o, o, sizeof s->o);
        s->nf = nf;
        s->tc = tc;
        s->nm = nm;
        s->moff = moff;
        s->w = w;
        s->out = out;
        s->p_lo = (int)((long)o[0] * t / threads);
        s->p_hi = (int)((long)o[0] * (t + 1) / threads);
        if (t > 0) pthread_create(&th[t], NULL, score_rows, s);
    }
    score_rows(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    free(moff);
    free(w);
}

int ccwo3_score_map(const int32_t* ti_counts, const int32_t* cdims, int nf, const int32_t* or_counts,
                    const uint8_t* mask, int tc, int64_t* out) {
    if (tc < 1 || tc > cdims[0] || tc > cdims[1] || tc > cdims[2])
        return fail(E_DIMENSION, "template %d larger than TI coefficients", tc);
    const int c[3] = {cdims[0], cdims[1], cdims[2]};
    score_map(ti_counts, c, nf, tc, or_counts, mask, 1, out);
    return 0;
}

/* ------------------------------------------------------------ plan ------- */
static int padded_extent(int sg, int t, int stride) { /* simulator.hpp:125-131 */
    if (sg == t) return t;
    const int steps = (sg - t + stride - 1) / stride;
    return t + steps * stride;
}

typedef struct {
    int corner, order;
    int work[3];
    int n[3];          /* placements per axis */
    int* pos[3];       /* traversal-ordered positions per axis */
    int count;
} plan3;

static void plan_free(plan3* p) {
    for (int a = 0; a < 3; ++a) free(p->pos[a]);
}

static void make_plan(const ccwo3_config* c, mt64* rng, plan3* p) { /* simulator.hpp:148-190 */
    const int t = c->template_size, stride = t - c->overlap;
    p->corner = (int)bounded(rng, 8);
    p->order = (int)bounded(rng, 6);
    p->count = 1;
    for (int a = 0; a < 3; ++a) {
        p->work[a] = padded_extent(c->sg[a], t, stride);
        p->n[a] = (p->work[a] - t) / stride + 1;
        p->pos[a] = malloc(sizeof(int) * p->n[a]);
        const int asc = !((p->corner >> a) & 1);
        for (int k = 0; k < p->n[a]; ++k) p->pos[a][asc ? k : p->n[a] - 1 - k] = k * stride;
        p->count *= p->n[a];
    }
}

/* placement k (raster order) -> traversal index per axis */
static void plan_index(const plan3* p, int k, int* idx) {
    const int* ord = ccwo3_orders[p->order];
    const int ni = p->n[ord[2]], nm = p->n[ord[1]];
    idx[ord[2]] = k % ni;
    idx[ord[1]] = (k / ni) % nm;
    idx[ord[0]] = k / (ni * nm);
}

int ccwo3_plan(const ccwo3_config* cfg, uint64_t seed, int* corner, int* order, int32_t* work,
               int32_t* origins, int32_t* shapes, int capacity, int* count) {
    int e = validate_cfg(cfg);
    if (e) return e;
    mt64 rng;
    mt_seed(&rng, seed);
    plan3 p;
    make_plan(cfg, &rng, &p);
    *corner = p.corner;
    *order = p.order;
    for (int a = 0; a < 3; ++a) work[a] = p.work[a];
    *count = p.count;
    for (int k = 0; k < p.count && k < capacity; ++k) {
        int idx[3];
        plan_index(&p, k, idx);
        int sh = 0;
        for (int a = 0; a < 3; ++a) {
            origins[3 * k + a] = p.pos[a][idx[a]];
            if (idx[a] > 0) sh |= 1 << a;
        }
        shapes[k] = sh;
    }
    plan_free(&p);
    return 0;
}

/* ------------------------------------------------------- simulation ------ */
typedef struct {
    int64_t s;
    int p;
} cand;

int ccwo3_simulate_one(const uint8_t* ti, const int32_t* ti_dims, int nf, const ccwo3_config* cfg,
                       const int32_t* hd, int n_hd, uint64_t seed, int threads, uint8_t* out,
                       ccwo3_diag* diag, int32_t* chosen) {
    int e = ccwo3_validate(cfg, ti_dims, nf, hd, n_hd);
    if (e) return e;
    const int J = cfg->dwt_level, B = 1 << J, T = cfg->template_size, OV = cfg->overlap;
    const int tc = T >> J, nt3 = tc * tc * tc;
    int used[3], c[3], o[3];
    for (int a = 0; a < 3; ++a) {
        used[a] = ti_dims[a] / B * B;
        c[a] = used[a] / B;
        o[a] = c[a] - tc + 1;
    }
    const size_t ncoarse = (size_t)c[0] * c[1] * c[2];
    const int npos = o[0] * o[1] * o[2];
    int32_t* counts = malloc(sizeof(int32_t) * ncoarse * nf);
    e = ccwo3_block_counts(ti, ti_dims, nf, J, counts);
    if (e) {
        free(counts);
        return e;
    }
    mt64 rng;
    mt_seed(&rng, seed);
    plan3 p;
    make_plan(cfg, &rng, &p);
    const size_t W1 = (size_t)p.work[1], W2 = (size_t)p.work[2];
    const size_t wn = (size_t)p.work[0] * W1 * W2;
    uint8_t* work = calloc(wn, 1);
    uint8_t* sim = calloc(wn, 1);
    int32_t* n = malloc(sizeof(int32_t) * (size_t)nt3 * nf);
    uint8_t* mask = malloc(nt3);
    int64_t* scores = malloc(sizeof(int64_t) * (size_t)npos);
    const int K = cfg->candidates < npos ? cfg->candidates : npos;
    cand* top = malloc(sizeof(cand) * (K + 1));
    int32_t* hdl = malloc(sizeof(int32_t) * 4 * (n_hd > 0 ? n_hd : 1));
    int rc = 0;
    for (int k = 0; k < p.count && !rc; ++k) {
        int idx[3], P[3], sh = 0, fr[3];
        plan_index(&p, k, idx);
        for (int a = 0; a < 3; ++a) {
            P[a] = p.pos[a][idx[a]];
            if (idx[a] > 0) sh |= 1 << a;
        }
        if (sh == 0) { /* simulator.hpp:450-453: random block-aligned TI patch */
            for (int a = 0; a < 3; ++a) fr[a] = (int)bounded(&rng, (uint64_t)((used[a] - T) / B + 1)) * B;
        } else {
            /* extract_or + coarse counts (simulator.hpp:225-272) */
            memset(n, 0, sizeof(int32_t) * (size_t)nt3 * nf);
            memset(mask, 0, nt3);
            int partial = 0;
            for (int m0 = 0; m0 < tc; ++m0)
                for (int m1 = 0; m1 < tc; ++m1)
                    for (int m2 = 0; m2 < tc; ++m2) {
                        const int m = (m0 * tc + m1) * tc + m2;
                        int in = 0, tot = 0;
                        for (int x0 = m0 * B; x0 < m0 * B + B; ++x0)
                            for (int x1 = m1 * B; x1 < m1 * B + B; ++x1)
                                for (int x2 = m2 * B; x2 < m2 * B + B; ++x2) {
                                    const int x[3] = {x0, x1, x2};
                                    int sup = 0;
                                    for (int a = 0; a < 3; ++a)
                                        if ((sh >> a) & 1) {
                                            const int asc = !((p.corner >> a) & 1);
                                            if (asc ? x[a] < OV : x[a] >= T - OV) sup = 1;
                                        }
                                    ++tot;
                                    if (!sup) continue;
                                    ++in;
                                    const size_t g = ((size_t)(P[0] + x0) * W1 + (P[1] + x1)) * W2 + (P[2] + x2);
                                    if (!sim[g]) {
                                        rc = fail(E_ERROR, "overlap cell (%d, %d, %d) not yet simulated", P[0] + x0,
                                                  P[1] + x1, P[2] + x2);
                                        goto done;
                                    }
                                    n[(size_t)work[g] * nt3 + m] += 1;
                                }
                        if (in) mask[m] = 1;
                        if (in && in != tot) partial = 1;
                    }
            if (partial && !cfg->any_support) { /* simulator.hpp:266-267 */
                rc = fail(E_STRUCTURE, "mask not aligned to 2^dwt_level blocks");
                goto done;
            }
            score_map(counts, c, nf, tc, n, mask, threads, scores);
            /* top_k (matcher.hpp:177-204) */
            int nt = 0;
            for (int q = 0; q < npos; ++q) {
                const int64_t s = scores[q];
                if (nt == K && s <= top[nt - 1].s) continue;
                int at = nt;
                while (at > 0 && top[at - 1].s < s) --at;
                memmove(top + at + 1, top + at, sizeof(cand) * (nt - at));
                top[at].s = s;
                top[at].p = q;
                if (nt < K) ++nt;
            }
            /* hard data under the footprint (simulator.hpp:467-473) */
            int nl = 0;
            for (int i = 0; i < n_hd; ++i) {
                const int* d = hd + 4 * i;
                if (d[0] >= P[0] && d[0] < P[0] + T && d[1] >= P[1] && d[1] < P[1] + T && d[2] >= P[2] &&
                    d[2] < P[2] + T) {
                    hdl[4 * nl] = d[0] - P[0];
                    hdl[4 * nl + 1] = d[1] - P[1];
                    hdl[4 * nl + 2] = d[2] - P[2];
                    hdl[4 * nl + 3] = d[3];
                    ++nl;
                }
            }
            int pick = 0;
            if (nl > 0) { /* select_conditional (matcher.hpp:222-241) */
                int best = 0, best_m = nl + 1;
                for (int ci = 0; ci < nt; ++ci) {
                    const int q = top[ci].p;
                    const int q0 = q / (o[1] * o[2]), q1 = (q / o[2]) % o[1], q2 = q % o[2];
                    int mm = 0;
                    for (int i = 0; i < nl; ++i) {
                        const size_t g = ((size_t)(q0 * B + hdl[4 * i]) * ti_dims[1] + (q1 * B + hdl[4 * i + 1])) *
                                             ti_dims[2] + (q2 * B + hdl[4 * i + 2]);
                        if (ti[g] != hdl[4 * i + 3]) ++mm;
                    }
                    if (mm == 0) {
                        best = ci;
                        break;
                    }
                    if (mm < best_m) {
                        best_m = mm;
                        best = ci;
                    }
                }
                pick = best;
            } else { /* select_unconditional (matcher.hpp:207-211) */
                pick = (int)bounded(&rng, (uint64_t)nt);
            }
            const int q = top[pick].p;
            fr[0] = q / (o[1] * o[2]) * B;
            fr[1] = (q / o[2]) % o[1] * B;
            fr[2] = q % o[2] * B;
        }
        /* crop + paste_into (grid.hpp:172-230, simulator.hpp:483-493) */
        for (int x0 = 0; x0 < T; ++x0)
            for (int x1 = 0; x1 < T; ++x1) {
                const size_t g = ((size_t)(P[0] + x0) * W1 + (P[1] + x1)) * W2 + P[2];
                const size_t s = ((size_t)(fr[0] + x0) * ti_dims[1] + (fr[1] + x1)) * ti_dims[2] + fr[2];
                memcpy(work + g, ti + s, T);
                memset(sim + g, 1, T);
            }
        if (chosen)
            for (int a = 0; a < 3; ++a) chosen[3 * k + a] = fr[a];
    }
done:
    if (!rc) {
        int mism = 0; /* simulator.hpp:506-513 */
        for (int i = 0; i < n_hd; ++i) {
            const int* d = hd + 4 * i;
            const size_t g = ((size_t)d[0] * W1 + d[1]) * W2 + d[2];
            if (work[g] != d[3]) ++mism;
            work[g] = (uint8_t)d[3];
        }
        for (int i0 = 0; i0 < cfg->sg[0]; ++i0) /* crop (simulator.hpp:515) */
            for (int i1 = 0; i1 < cfg->sg[1]; ++i1)
                memcpy(out + ((size_t)i0 * cfg->sg[1] + i1) * cfg->sg[2], work + ((size_t)i0 * W1 + i1) * W2,
                       cfg->sg[2]);
        if (diag) {
            diag->seed = seed;
            diag->corner = p.corner;
            diag->order = p.order;
            for (int a = 0; a < 3; ++a) diag->work[a] = p.work[a];
            diag->placement_count = p.count;
            diag->hard_data_count = n_hd;
            diag->pre_overwrite_mismatches = mism;
        }
    }
    plan_free(&p);
    free(counts);
    free(work);
    free(sim);
    free(n);
    free(mask);
    free(scores);
    free(top);
    free(hdl);
    return rc;
}

/* simulator.hpp:523-566 */
typedef struct {
    const uint8_t* ti;
    const int32_t* dims;
    int nf;
    const ccwo3_config* cfg;
    const int32_t* hd;
    int n_hd;
    uint8_t* out;
    ccwo3_diag* diags;
    int next, err;
    char msg[512];
    pthread_mutex_t mu;
} ens_state;

static void* ens_worker(void* arg) {
    ens_state* s = (ens_state*)arg;
    const size_t sgn = (size_t)s->cfg->sg[0] * s->cfg->sg[1] * s->cfg->sg[2];
    for (;;) {
        pthread_mutex_lock(&s->mu);
        const int r = s->err ? s->cfg->n_realizations : s->next++;
        pthread_mutex_unlock(&s->mu);
        if (r >= s->cfg->n_realizations) return NULL;
        const int e = ccwo3_simulate_one(s->ti, s->dims, s->nf, s->cfg, s->hd, s->n_hd,
                                         mix64(s->cfg->master_seed, (uint64_t)r + 1), 1, s->out + sgn * r,
                                         s->diags ? &s->diags[r] : NULL, NULL);
        if (e) {
            pthread_mutex_lock(&s->mu);
            if (!s->err) {
                s->err = e;
                snprintf(s->msg, sizeof s->msg, "%s", g_err);
            }
            pthread_mutex_unlock(&s->mu);
        }
    }
}

int ccwo3_simulate_ensemble(const uint8_t* ti, const int32_t* ti_dims, int nf, const ccwo3_config* cfg,
                            const int32_t* hd, int n_hd, int workers, uint8_t* out, ccwo3_diag* diags) {
    int e = ccwo3_validate(cfg, ti_dims, nf, hd, n_hd);
    if (e) return e;
    ens_state s = {ti, ti_dims, nf, cfg, hd, n_hd, out, diags, 0, 0, {0}, PTHREAD_MUTEX_INITIALIZER};
    if (workers < 1) workers = 1;
    if (workers > cfg->n_realizations) workers = cfg->n_realizations;
    pthread_t* th = malloc(sizeof(pthread_t) * workers);
    for (int w = 1; w < workers; ++w) pthread_create(&th[w], NULL, ens_worker, &s);
    ens_worker(&s);
    for (int w = 1; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
    if (s.err) return fail(s.err, "%s", s.msg);
    return 0;
}
