/*
 * ccw_metrics_oracle.c -- CPU restatement of the reference's validation
 * metrics (proj/include/ccwsim/metrics.hpp:68-437), the consumers of the
 * simulated ensembles.  TEST INFRASTRUCTURE ONLY (tests/ and bench.py's CPU
 * legs): the product never links it.
 *
 * metrics.hpp includes Eigen (:13) for its MDS step, so the reference header
 * cannot be compiled here; this restatement follows its loops line by line
 * and is pinned on the reference's own known answers (proj/tests/
 * test_metrics.cpp) restated in tests/test_metrics_cpu.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* metrics.hpp:68-112.  gamma[h-1], h = 1..max_lag; returns facies_present. */
int ccwm_variogram(const uint8_t* g, int h, int w, int facies, int direction, int max_lag, double* gamma) {
    int present = 0;
    for (long i = 0; i < (long)h * w && !present; ++i) present = g[i] == facies;
    for (int lag = 1; lag <= max_lag; ++lag) {
        int64_t pairs = 0, sum_sq = 0;
        if (direction == 0) { /* east_west */
            for (int r = 0; r < h; ++r)
                for (int c = 0; c + lag < w; ++c) {
                    const int a = g[(long)r * w + c] == facies, b = g[(long)r * w + c + lag] == facies;
                    sum_sq += (a - b) * (a - b);
                    ++pairs;
                }
        } else {
            for (int r = 0; r + lag < h; ++r)
                for (int c = 0; c < w; ++c) {
                    const int a = g[(long)r * w + c] == facies, b = g[(long)(r + lag) * w + c] == facies;
                    sum_sq += (a - b) * (a - b);
                    ++pairs;
                }
        }
        gamma[lag - 1] = pairs > 0 ? 0.5 * (double)sum_sq / (double)pairs : 0.0;
    }
    return present;
}

/* metrics.hpp:116-154: 4-connected labels (union-find, smaller root wins). */
static int find(int* parent, int x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

static void label_components(const uint8_t* g, int h, int w, int facies, int* labels) {
    const long n = (long)h * w;
    int* parent = malloc(sizeof(int) * n);
    for (long i = 0; i < n; ++i) parent[i] = (int)i;
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            if (g[(long)r * w + c] != facies) continue;
            const int idx = r * w + c;
            if (c + 1 < w && g[idx + 1] == facies) {
                int a = find(parent, idx), b = find(parent, idx + 1);
                if (a != b) parent[a > b ? a : b] = a < b ? a : b;
            }
            if (r + 1 < h && g[idx + w] == facies) {
                int a = find(parent, idx), b = find(parent, idx + w);
                if (a != b) parent[a > b ? a : b] = a < b ? a : b;
            }
        }
    for (long i = 0; i < n; ++i) labels[i] = g[i] == facies ? find(parent, (int)i) : -1;
    free(parent);
}

/* metrics.hpp:158-205.  prob[h-1] = NaN where no same-facies pair exists. */
void ccwm_connectivity(const uint8_t* g, int h, int w, int facies, int direction, int max_lag, double* prob) {
    int* lab = malloc(sizeof(int) * (size_t)h * w);
    label_components(g, h, w, facies, lab);
    for (int lag = 1; lag <= max_lag; ++lag) {
        int64_t both = 0, conn = 0;
        if (direction == 0) {
            for (int r = 0; r < h; ++r)
                for (int c = 0; c + lag < w; ++c) {
                    const int la = lab[(long)r * w + c], lb = lab[(long)r * w + c + lag];
                    if (la >= 0 && lb >= 0) {
                        ++both;
                        conn += la == lb;
                    }
                }
        } else {
            for (int r = 0; r + lag < h; ++r)
                for (int c = 0; c < w; ++c) {
                    const int la = lab[(long)r * w + c], lb = lab[(long)(r + lag) * w + c];
                    if (la >= 0 && lb >= 0) {
                        ++both;
                        conn += la == lb;
                    }
                }
        }
        prob[lag - 1] = both > 0 ? (double)conn / (double)both : NAN;
    }
    free(lab);
}

/* metrics.hpp:208-227 */
void ccwm_ensemble_average(const uint8_t* grids, int n, int h, int w, int facies, double* out) {
    const long cells = (long)h * w;
    for (long i = 0; i < cells; ++i) out[i] = 0.0;
    for (int r = 0; r < n; ++r)
        for (long i = 0; i < cells; ++i)
            if (grids[(long)r * cells + i] == facies) out[i] += 1.0;
    for (long i = 0; i < cells; ++i) out[i] /= (double)n;
}

/* metrics.hpp:230-254: the w x w windows at `stride`, keys = row-major codes.
 * keys (capacity windows * win^2 bytes) get the distinct keys in
 * lexicographic order, counts their multiplicity; returns the distinct count
 * (total = number of windows in *total). */
static int g_kw;
static int key_cmp(const void* a, const void* b) { return memcmp(a, b, (size_t)g_kw); }

int ccwm_pattern_histogram(const uint8_t* g, int h, int w, int win, int stride, uint8_t* keys, uint64_t* counts,
                           uint64_t* total) {
    const int kw = win * win;
    long nwin = 0;
    for (int top = 0; top + win <= h; top += stride)
        for (int left = 0; left + win <= w; left += stride) ++nwin;
    uint8_t* all = malloc((size_t)(nwin > 0 ? nwin : 1) * kw);
    long k = 0;
    for (int top = 0; top + win <= h; top += stride)
        for (int left = 0; left + win <= w; left += stride, ++k)
            for (int r = 0; r < win; ++r) memcpy(all + k * kw + r * win, g + (long)(top + r) * w + left, (size_t)win);
    g_kw = kw;
    qsort(all, (size_t)nwin, (size_t)kw, key_cmp);
    int nd = 0;
    for (long i = 0; i < nwin; ++i) {
        if (i > 0 && memcmp(all + i * kw, all + (i - 1) * kw, (size_t)kw) == 0) {
            ++counts[nd - 1];
            continue;
        }
        memcpy(keys + (size_t)nd * kw, all + i * kw, (size_t)kw);
        counts[nd++] = 1;
    }
    *total = (uint64_t)nwin;
    free(all);
    return nd;
}

/* metrics.hpp:258-284 over two sorted histograms (sum in key order). */
double ccwm_js_divergence(const uint8_t* pk, const uint64_t* pc, int np, uint64_t pt, const uint8_t* qk,
                          const uint64_t* qc, int nq, uint64_t qt, int kw) {
    double sum = 0.0;
    int j = 0;
    for (int i = 0; i < np; ++i) {
        while (j < nq && memcmp(qk + (size_t)j * kw, pk + (size_t)i * kw, (size_t)kw) < 0) ++j;
        const double pp = (double)pc[i] / (double)pt;
        const double qq = (j < nq && memcmp(qk + (size_t)j * kw, pk + (size_t)i * kw, (size_t)kw) == 0)
                              ? (double)qc[j] / (double)qt
                              : 0.0;
        sum += 0.5 * pp * log2(2.0 * pp / (pp + qq));
    }
    int i = 0;
    for (int jj = 0; jj < nq; ++jj) {
        while (i < np && memcmp(pk + (size_t)i * kw, qk + (size_t)jj * kw, (size_t)kw) < 0) ++i;
        const double qq = (double)qc[jj] / (double)qt;
        const double pp = (i < np && memcmp(pk + (size_t)i * kw, qk + (size_t)jj * kw, (size_t)kw) == 0)
                              ? (double)pc[i] / (double)pt
                              : 0.0;
        sum += 0.5 * qq * log2(2.0 * qq / (pp + qq));
    }
    return sum < 0.0 ? 0.0 : (sum > 1.0 ? 1.0 : sum);
}

/* metrics.hpp:288-311: block-majority downsampling, ties to the lowest code. */
void ccwm_downsample_majority(const uint8_t* g, int h, int w, int nf, int factor, uint8_t* out) {
    const int oh = h / factor, ow = w / factor;
    int* cnt = malloc(sizeof(int) * (size_t)nf);
    for (int i = 0; i < oh; ++i)
        for (int j = 0; j < ow; ++j) {
            memset(cnt, 0, sizeof(int) * (size_t)nf);
            for (int r = 0; r < factor; ++r)
                for (int c = 0; c < factor; ++c) ++cnt[g[(long)(i * factor + r) * w + j * factor + c]];
            int best = 0;
            for (int f = 1; f < nf; ++f)
                if (cnt[f] > cnt[best]) best = f;
            out[(long)i * ow + j] = (uint8_t)best;
        }
    free(cnt);
}

/* metrics.hpp:318-384 (ANODI without the MDS step).  out: levels x 8
 * doubles (between_a, between_b, within_a, within_b, d_between, d_within,
 * ratio, weight).  Returns 0, 5 (EmptyInput), 2 (Dimension), 3 (Structure)
 * or 8 (Degeneracy). */
typedef struct {
    uint8_t* keys;
    uint64_t* counts;
    int n;
    uint64_t total;
} hist_t;

static hist_t make_hist(const uint8_t* g, int h, int w, int nf, int factor, int win) {
    const int oh = h / factor, ow = w / factor;
    uint8_t* d = malloc((size_t)oh * ow);
    if (factor == 1)
        memcpy(d, g, (size_t)h * w);
    else
        ccwm_downsample_majority(g, h, w, nf, factor, d);
    const long nwin = (long)(oh - win + 1) * (ow - win + 1);
    hist_t r;
    r.keys = malloc((size_t)(nwin > 0 ? nwin : 1) * win * win);
    r.counts = malloc(sizeof(uint64_t) * (size_t)(nwin > 0 ? nwin : 1));
    r.n = nwin > 0 ? ccwm_pattern_histogram(d, oh, ow, win, 1, r.keys, r.counts, &r.total) : 0;
    if (nwin <= 0) r.total = 0;
    free(d);
    return r;
}

int ccwm_anodi(const uint8_t* ga, int na, const uint8_t* gb, int nb, int h, int w, const uint8_t* ti, int th,
               int tw, int nf, int levels, int win, const double* weights, double* out, double* aggregate) {
    if (na < 2 || nb < 2) return 5;
    if (levels < 1) return 2;
    const int kw = win * win;
    *aggregate = 0.0;
    for (int p = 1; p <= levels; ++p) {
        const int factor = 1 << (p - 1);
        hist_t* ha = malloc(sizeof(hist_t) * na);
        hist_t* hb = malloc(sizeof(hist_t) * nb);
        for (int i = 0; i < na; ++i) ha[i] = make_hist(ga + (size_t)i * h * w, h, w, nf, factor, win);
        for (int i = 0; i < nb; ++i) hb[i] = make_hist(gb + (size_t)i * h * w, h, w, nf, factor, win);
        hist_t ht = make_hist(ti, th, tw, nf, factor, win);
        double s = 0.0;
        size_t pairs = 0;
        for (int i = 0; i < na; ++i)
            for (int j = i + 1; j < na; ++j, ++pairs)
                s += ccwm_js_divergence(ha[i].keys, ha[i].counts, ha[i].n, ha[i].total, ha[j].keys, ha[j].counts,
                                        ha[j].n, ha[j].total, kw);
        const double between_a = s / (double)pairs;
        s = 0.0;
        pairs = 0;
        for (int i = 0; i < nb; ++i)
            for (int j = i + 1; j < nb; ++j, ++pairs)
                s += ccwm_js_divergence(hb[i].keys, hb[i].counts, hb[i].n, hb[i].total, hb[j].keys, hb[j].counts,
                                        hb[j].n, hb[j].total, kw);
        const double between_b = s / (double)pairs;
        s = 0.0;
        for (int i = 0; i < na; ++i)
            s += ccwm_js_divergence(ha[i].keys, ha[i].counts, ha[i].n, ha[i].total, ht.keys, ht.counts, ht.n, ht.total,
                                    kw);
        const double within_a = s / (double)na;
        s = 0.0;
        for (int i = 0; i < nb; ++i)
            s += ccwm_js_divergence(hb[i].keys, hb[i].counts, hb[i].n, hb[i].total, ht.keys, ht.counts, ht.n, ht.total,
                                    kw);
        const double within_b = s / (double)nb;
        for (int i = 0; i < na; ++i) {
            free(ha[i].keys);
            free(ha[i].counts);
        }
        for (int i = 0; i < nb; ++i) {
            free(hb[i].keys);
            free(hb[i].counts);
        }
        free(ha);
        free(hb);
        free(ht.keys);
        free(ht.counts);
        double* o = out + (size_t)(p - 1) * 8;
        o[0] = between_a;
        o[1] = between_b;
        o[2] = within_a;
        o[3] = within_b;
        o[7] = weights ? weights[p - 1] : 1.0 / levels;
        if (within_a == 0.0 || within_b == 0.0 || between_b == 0.0) return 8;
        o[4] = between_a / between_b;
        o[5] = within_a / within_b;
        o[6] = o[4] / o[5];
        *aggregate += o[7] * o[6];
    }
    return 0;
}
