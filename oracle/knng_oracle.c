/*
 * knng_oracle.c -- TEST INFRASTRUCTURE ONLY.  See knng_oracle.h.
 *
 * Plain single-threaded C99, compiled with -O2 -ffp-contract=off (no fast
 * math) so every float operation is the one written here.  Nothing is
 * blocked, fused or reordered beyond what the paper's algorithms state;
 * every function cites the passage it follows.
 */
#include "knng_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define KEY(d, id) ((((uint64_t)f2u(d)) << 32) | (uint64_t)(uint32_t)(id))
#define KEY_ID(key) ((uint32_t)((key) & 0xFFFFFFFFull))

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static float key_dist(uint64_t key) { return u2f((uint32_t)(key >> 32)); }

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (D31).  Round: (c0,c1,c2,c3) ->                        */
/*   (hi(M1*c2) ^ c1 ^ k0, lo(M1*c2), hi(M0*c0) ^ c3 ^ k1, lo(M0*c0))   */
/* with M0 = 0xD2511F53, M1 = 0xCD9E8D57; key bumped by the Weyl        */
/* constants (0x9E3779B9, 0xBB67AE85) between rounds.                   */
/* ------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                       uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t orc_uniform(const uint32_t out[4], uint64_t N) {
    uint64_t r = ((uint64_t)out[1] << 32) | (uint64_t)out[0];
    return (uint64_t)(((unsigned __int128)r * (unsigned __int128)N) >> 64);
}

static void philox_words(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                         uint64_t seed, uint32_t out[4]) {
    uint32_t ctr[4] = {w0, w1, w2, w3};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------ */
/* Metric ("l2-norm"; D4 squared; D5 canonical order; D6 cosine)  */
/* ------------------------------------------------------------------ */
typedef struct {
    const void* X;
    int dtype;
    int64_t n;
    int d;
    int metric;
    float* Xn; /* cosine: pre-normalised rows */
} dataset;

static int ds_open(dataset* ds, const void* X, int dtype, int64_t n, int d,
                   int metric) {
    ds->X = X; ds->dtype = dtype; ds->n = n; ds->d = d; ds->metric = metric;
    ds->Xn = NULL;
    if (dtype != ORC_F32 && dtype != ORC_U8) return ORC_E_USAGE;
    if (metric != ORC_L2SQ && metric != ORC_COSINE && metric != ORC_CHI2) return ORC_E_USAGE;
    if (metric == ORC_CHI2 && dtype == ORC_F32) {
        /* chi-square needs non-negative components (D39) */
        const float* F = (const float*)X;
        for (int64_t i = 0; i < n * (int64_t)d; ++i)
            if (!(F[i] >= 0.0f)) return ORC_E_DOMAIN;
    }
    if (metric == ORC_COSINE) {
        if (dtype != ORC_F32) return ORC_E_USAGE;
        const float* F = (const float*)X;
        ds->Xn = (float*)malloc((size_t)n * (size_t)d * sizeof(float));
        if (!ds->Xn) return ORC_E_NOMEM;
        for (int64_t i = 0; i < n; ++i) {
            const float* x = F + (size_t)i * d;
            float acc = 0.0f;
            for (int j = 0; j < d; ++j) acc = fmaf(x[j], x[j], acc);
            if (!(acc > 0.0f)) { free(ds->Xn); ds->Xn = NULL; return ORC_E_DOMAIN; }
            float r = 1.0f / sqrtf(acc);
            for (int j = 0; j < d; ++j) ds->Xn[(size_t)i * d + j] = x[j] * r;
        }
    }
    return ORC_OK;
}

static void ds_close(dataset* ds) { free(ds->Xn); ds->Xn = NULL; }

/* chi-square ("K-Square"), D39: terms (x_i - y_i)^2 / (x_i + y_i) in
 * dimension order; q = t / s (0 when s = 0), acc = fmaf(q, t, acc). */
static float chi2_term(float x, float y, float acc) {
    float t = x - y;
    float s = x + y;
    float q = (s > 0.0f) ? t / s : 0.0f;
    return fmaf(q, t, acc);
}

static float ds_dist(const dataset* ds, int64_t a, int64_t b) {
    const int d = ds->d;
    if (ds->metric == ORC_CHI2) {
        float acc = 0.0f;
        if (ds->dtype == ORC_U8) {
            const uint8_t* x = (const uint8_t*)ds->X + (size_t)a * d;
            const uint8_t* y = (const uint8_t*)ds->X + (size_t)b * d;
            for (int i = 0; i < d; ++i) acc = chi2_term((float)x[i], (float)y[i], acc);
        } else {
            const float* x = (const float*)ds->X + (size_t)a * d;
            const float* y = (const float*)ds->X + (size_t)b * d;
            for (int i = 0; i < d; ++i) acc = chi2_term(x[i], y[i], acc);
        }
        return acc;
    }
    if (ds->metric == ORC_COSINE) {
        const float* x = ds->Xn + (size_t)a * d;
        const float* y = ds->Xn + (size_t)b * d;
        float s = 0.0f;
        for (int i = 0; i < d; ++i) s = fmaf(x[i], y[i], s);
        float r = 1.0f - s;
        return (r > 0.0f) ? r : 0.0f;
    }
    if (ds->dtype == ORC_U8) {
        const uint8_t* x = (const uint8_t*)ds->X + (size_t)a * d;
        const uint8_t* y = (const uint8_t*)ds->X + (size_t)b * d;
        int64_t acc = 0;
        for (int i = 0; i < d; ++i) {
            int64_t t = (int64_t)x[i] - (int64_t)y[i];
            acc += t * t;
        }
        return (float)acc;
    }
    const float* x = (const float*)ds->X + (size_t)a * d;
    const float* y = (const float*)ds->X + (size_t)b * d;
    float acc = 0.0f;
    for (int i = 0; i < d; ++i) {
        float t = x[i] - y[i];
        acc = fmaf(t, t, acc);
    }
    return acc;
}

float orc_distance(const void* X, int dtype, int64_t n, int d, int metric,
                   int64_t a, int64_t b) {
    dataset ds;
    if (ds_open(&ds, X, dtype, n, d, metric) != ORC_OK) return -1.0f;
    float r = ds_dist(&ds, a, b);
    ds_close(&ds);
    return r;
}

/* ------------------------------------------------------------------ */
/* Process-wide oracle options (test infrastructure)                    */
/* ------------------------------------------------------------------ */
static int g_update_mode = ORC_UPDATE_SELECTIVE;
static int g_seg_size = 32;

int orc_set_option(const char* name, int value) {
    if (strcmp(name, "update") == 0) {
        if (value != ORC_UPDATE_SELECTIVE && value != ORC_UPDATE_FULL) return ORC_E_USAGE;
        g_update_mode = value;
        return ORC_OK;
    }
    if (strcmp(name, "segment_size") == 0) {
        if (value < 1) return ORC_E_USAGE;
        g_seg_size = value;
        return ORC_OK;
    }
    return ORC_E_USAGE;
}

/* segments of a k-list ("divided into k / 32 segments", D18/D40):
 * s = k / seg for k >= 2 seg (k a multiple of seg), else 1 */
int orc_segments(int k) {
    if (k >= 2 * g_seg_size) return (k % g_seg_size == 0) ? k / g_seg_size : -1;
    return 1;
}

/* ------------------------------------------------------------------ */
/* Bounded sorted k-NN list (D16)                          */
/* ------------------------------------------------------------------ */
static int list_has_id(const uint64_t* L, int k, uint32_t id) {
    for (int j = 0; j < k; ++j)
        if (L[j] != ORC_SENTINEL && KEY_ID(L[j]) == id) return 1;
    return 0;
}

/* InsertIntoNNList(G[u], v, d): accept iff key < current maximum and id not
 * already in the list; the farthest entry is evicted; the new entry is NEW.
 * Returns 1 if inserted.
 * Segmented list (s > 1, D40): the list is kept as the sorted union
 * of its s segments; entry id v belongs to segment v % s, every segment
 * holds k / s entries.  The candidate competes only with its own segment:
 * accept iff key < that segment's maximum and v is not in the list (it
 * could only be in its own segment); that segment's maximum is evicted. */
static int list_insert_seg(uint64_t* L, uint8_t* F, int k, int s, uint64_t key) {
    if (list_has_id(L, k, KEY_ID(key))) return 0;
    const uint32_t g = KEY_ID(key) % (uint32_t)s;
    int evict = -1; /* position of the segment's maximum (segments are full) */
    for (int j = k - 1; j >= 0; --j)
        if (L[j] != ORC_SENTINEL && KEY_ID(L[j]) % (uint32_t)s == g) { evict = j; break; }
    if (evict < 0 || !(key < L[evict])) return 0;
    for (int j = evict; j < k - 1; ++j) { L[j] = L[j + 1]; F[j] = F[j + 1]; } /* remove it */
    int pos = k - 1;
    while (pos > 0 && L[pos - 1] > key) {
        L[pos] = L[pos - 1];
        F[pos] = F[pos - 1];
        --pos;
    }
    L[pos] = key;
    F[pos] = 1;
    return 1;
}

static int list_insert(uint64_t* L, uint8_t* F, int k, uint64_t key) {
    if (!(key < L[k - 1])) return 0;
    if (list_has_id(L, k, KEY_ID(key))) return 0;
    int pos = k - 1;
    while (pos > 0 && L[pos - 1] > key) {
        L[pos] = L[pos - 1];
        F[pos] = F[pos - 1];
        --pos;
    }
    L[pos] = key;
    F[pos] = 1;
    return 1;
}

int orc_list_insert(uint64_t* list, uint8_t* flags, int k, uint64_t key) {
    return list_insert(list, flags, k, key);
}

int orc_list_insert_seg(uint64_t* list, uint8_t* flags, int k, int s, uint64_t key) {
    if (s < 1 || k % s) return -1;
    return list_insert_seg(list, flags, k, s, key);
}

void orc_pair_index(int64_t t, int64_t* u, int64_t* v) {
    double uu = ceil(sqrt(2.0 * (double)t + 2.25) - 0.5);
    *u = (int64_t)uu;
    *v = t - (*u) * (*u - 1) / 2;
}

/* sort (key, flag) pairs ascending by key: insertion sort (k is small) */
static void sort_keys_flags(uint64_t* L, uint8_t* F, int k) {
    for (int i = 1; i < k; ++i) {
        uint64_t key = L[i];
        uint8_t f = F ? F[i] : 0;
        int j = i;
        while (j > 0 && L[j - 1] > key) {
            L[j] = L[j - 1];
            if (F) F[j] = F[j - 1];
            --j;
        }
        L[j] = key;
        if (F) F[j] = f;
    }
}

/* ------------------------------------------------------------------ */
/* Init: Alg. 1 lines 1-4 with D1 (k objects), D2 (distinct,  */
/* != s, Philox rejection), D3 (sort by key), all NEW.          */
/* ------------------------------------------------------------------ */
static int init_list(const dataset* ds, int k, uint64_t seed, int64_t s,
                     uint64_t* L, uint8_t* F) {
    int64_t n = ds->n;
    const int nseg = orc_segments(k), per = k / nseg;
    uint32_t* chosen = (uint32_t*)malloc((size_t)k * sizeof(uint32_t));
    if (!chosen) return ORC_E_NOMEM;
    int cnt = 0;
    /* segment g (residue g mod nseg; one segment: all ids): per distinct
     * ids != s, drawn in counter order j from Philox(INIT, s, j | g << 24,
     * s >> 32) over the residue class without s (D2, D40) */
    for (int g = 0; g < nseg; ++g) {
        const int64_t M = (n - g + nseg - 1) / nseg;         /* ids = g mod nseg */
        const int self_in = (s % nseg) == g;
        const int start = cnt;
        for (uint32_t j = 0; cnt < start + per; ++j) {
            uint32_t out[4];
            philox_words(ORC_TAG_INIT, (uint32_t)s, j | ((uint32_t)g << 24),
                         (uint32_t)((uint64_t)s >> 32), seed, out);
            uint64_t r = orc_uniform(out, (uint64_t)(M - self_in));
            uint64_t v = (uint64_t)g + (uint64_t)nseg * r;
            if (self_in && v >= (uint64_t)s) v += (uint64_t)nseg;
            int dup = 0;
            for (int i = start; i < cnt; ++i)
                if (chosen[i] == (uint32_t)v) { dup = 1; break; }
            if (!dup) chosen[cnt++] = (uint32_t)v;
        }
    }
    for (int i = 0; i < k; ++i) {
        L[i] = KEY(ds_dist(ds, s, chosen[i]), chosen[i]);
        F[i] = 1;
    }
    sort_keys_flags(L, F, k);
    free(chosen);
    return ORC_OK;
}

int orc_init(const void* X, int dtype, int64_t n, int d, int metric, int k,
             uint64_t seed, uint64_t* keys, uint8_t* flags) {
    if (k < 1 || n <= k || d < 1) return ORC_E_USAGE;
    const int nseg = orc_segments(k);
    if (nseg < 1 || (nseg > 1 && n < (int64_t)k + nseg)) return ORC_E_USAGE;
    dataset ds;
    int rc = ds_open(&ds, X, dtype, n, d, metric);
    if (rc) return rc;
    for (int64_t s = 0; s < n && rc == ORC_OK; ++s)
        rc = init_list(&ds, k, seed, s, keys + (size_t)s * k, flags + (size_t)s * k);
    ds_close(&ds);
    return rc;
}

/* ------------------------------------------------------------------ */
/* ParallelSample                                           */
/* ------------------------------------------------------------------ */
typedef struct { uint32_t prio; uint32_t s; } rev_item;

static int cmp_rev(const void* a, const void* b) {
    const rev_item* x = (const rev_item*)a;
    const rev_item* y = (const rev_item*)b;
    if (x->prio != y->prio) return x->prio < y->prio ? -1 : 1;
    if (x->s != y->s) return x->s < y->s ? -1 : 1;
    return 0;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* G(v) = sort_unique(F(v) U c smallest-priority members of R(v)),
 * c = 2p - |F(v)|  (P:149 cap 2p counted with the forward samples, D8;
 * reverse edges from forward samples only, D9; priority D10). */
static int build_sample_lists(int64_t n, int p, uint32_t tag, uint32_t tword,
                              uint64_t seed, const uint32_t* Fw,
                              const int32_t* fc, uint32_t* G, int32_t* gc) {
    const int cap = 2 * p;
    int64_t* off = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!off) return ORC_E_NOMEM;
    for (int64_t s = 0; s < n; ++s)
        for (int i = 0; i < fc[s]; ++i) off[Fw[(size_t)s * p + i] + 1]++;
    for (int64_t v = 0; v < n; ++v) off[v + 1] += off[v];
    int64_t total = off[n];
    uint32_t* rsrc = (uint32_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(uint32_t));
    int64_t* fill = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    rev_item* items = NULL;
    size_t items_cap = 0;
    uint32_t* tmp = (uint32_t*)malloc((size_t)(cap + p + 1) * sizeof(uint32_t));
    if (!rsrc || !fill || !tmp) { free(off); free(rsrc); free(fill); free(tmp); return ORC_E_NOMEM; }
    for (int64_t s = 0; s < n; ++s)
        for (int i = 0; i < fc[s]; ++i) {
            uint32_t v = Fw[(size_t)s * p + i];
            rsrc[off[v] + fill[v]++] = (uint32_t)s;
        }
    int rc = ORC_OK;
    for (int64_t v = 0; v < n; ++v) {
        int64_t r = off[v + 1] - off[v];
        int c = cap - fc[v];
        int take = (r < c) ? (int)r : c;
        int len = 0;
        for (int i = 0; i < fc[v]; ++i) tmp[len++] = Fw[(size_t)v * p + i];
        if (r <= c) {
            for (int64_t i = 0; i < r; ++i) tmp[len++] = rsrc[off[v] + i];
        } else {
            if ((size_t)r > items_cap) {
                free(items);
                items_cap = (size_t)r;
                items = (rev_item*)malloc(items_cap * sizeof(rev_item));
                if (!items) { rc = ORC_E_NOMEM; break; }
            }
            for (int64_t i = 0; i < r; ++i) {
                uint32_t s = rsrc[off[v] + i];
                uint32_t out[4];
                philox_words(tag, tword, s, (uint32_t)v, seed, out);
                items[i].prio = out[0];
                items[i].s = s;
            }
            qsort(items, (size_t)r, sizeof(rev_item), cmp_rev);
            for (int i = 0; i < take; ++i) tmp[len++] = items[i].s;
        }
        qsort(tmp, (size_t)len, sizeof(uint32_t), cmp_u32);
        int u = 0;
        for (int i = 0; i < len; ++i)
            if (i == 0 || tmp[i] != tmp[i - 1]) G[(size_t)v * cap + u++] = tmp[i];
        gc[v] = u;
    }
    free(items); free(off); free(rsrc); free(fill); free(tmp);
    return rc;
}

int orc_sample(int64_t n, int k, int p, uint32_t tword, uint64_t seed,
               const uint64_t* keys, const uint8_t* flags,
               uint32_t* FN, int32_t* fnc, uint32_t* FO, int32_t* foc,
               uint32_t* Gn, int32_t* cn, uint32_t* Go, int32_t* co) {
    if (p < 1 || p >= k || n <= k) return ORC_E_USAGE;
    const int cap = 2 * p;
    int rc = ORC_E_NOMEM;
    uint32_t* fn = FN ? FN : (uint32_t*)malloc((size_t)n * p * sizeof(uint32_t));
    uint32_t* fo = FO ? FO : (uint32_t*)malloc((size_t)n * p * sizeof(uint32_t));
    int32_t* fnc_ = fnc ? fnc : (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* foc_ = foc ? foc : (int32_t*)malloc((size_t)n * sizeof(int32_t));
    uint32_t* gn = Gn ? Gn : (uint32_t*)malloc((size_t)n * cap * sizeof(uint32_t));
    uint32_t* go = Go ? Go : (uint32_t*)malloc((size_t)n * cap * sizeof(uint32_t));
    int32_t* cn_ = cn ? cn : (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* co_ = co ? co : (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!fn || !fo || !fnc_ || !foc_ || !gn || !go || !cn_ || !co_) goto done;

    /* Forward: "only the first p objects are sampled for either OLD
     * neighbors or NEW neighbors from one k-NN list" (D7). */
    for (int64_t s = 0; s < n; ++s) {
        int a = 0, b = 0;
        for (int j = 0; j < k; ++j) {
            uint64_t key = keys[(size_t)s * k + j];
            if (key == ORC_SENTINEL) continue;
            if (flags[(size_t)s * k + j]) {
                if (a < p) fn[(size_t)s * p + a++] = KEY_ID(key);
            } else {
                if (b < p) fo[(size_t)s * p + b++] = KEY_ID(key);
            }
        }
        fnc_[s] = a;
        foc_[s] = b;
    }
    /* Reverse append with cap 2p, then sort + dedup. */
    rc = build_sample_lists(n, p, ORC_TAG_REV_NEW, tword, seed, fn, fnc_, gn, cn_);
    if (rc) goto done;
    rc = build_sample_lists(n, p, ORC_TAG_REV_OLD, tword, seed, fo, foc_, go, co_);
    if (rc) goto done;
    /* D11: an id in both G_new(v) and G_old(v) stays NEW only. */
    for (int64_t v = 0; v < n; ++v) {
        const uint32_t* a = gn + (size_t)v * cap;
        uint32_t* b = go + (size_t)v * cap;
        int w = 0;
        for (int i = 0; i < co_[v]; ++i) {
            int in_new = 0;
            for (int j = 0; j < cn_[v]; ++j)
                if (a[j] == b[i]) { in_new = 1; break; }
            if (!in_new) b[w++] = b[i];
        }
        co_[v] = w;
    }
    rc = ORC_OK;
done:
    if (!FN) free(fn);
    if (!FO) free(fo);
    if (!fnc) free(fnc_);
    if (!foc) free(foc_);
    if (!Gn) free(gn);
    if (!Go) free(go);
    if (!cn) free(cn_);
    if (!co) free(co_);
    return rc;
}

/* ------------------------------------------------------------------ */
/* One iteration: Alg. 1 body                               */
/* ------------------------------------------------------------------ */
static int allowed_pair(int64_t boundary, uint32_t a, uint32_t b) {
    if (boundary < 0) return 1;
    return ((int64_t)a >= boundary) != ((int64_t)b >= boundary);
}

static void offer(uint64_t* keys, uint8_t* flags, int k, const uint8_t* tmask,
                  uint32_t target, uint64_t cand, orc_stats* st) {
    if (cand == ORC_SENTINEL) return; /* D15: (inf, inf) inserts nothing */
    st->candidates++;
    if (tmask && !tmask[target]) return;
    const int nseg = orc_segments(k);
    if (nseg > 1)
        list_insert_seg(keys + (size_t)target * k, flags + (size_t)target * k, k, nseg, cand);
    else
        list_insert(keys + (size_t)target * k, flags + (size_t)target * k, k, cand);
}

int orc_iterate(const void* X, int dtype, int64_t n, int d, int metric, int k,
                int p, uint32_t tword, uint64_t seed, int64_t boundary,
                uint64_t* keys, uint8_t* flags, const uint8_t* target_mask,
                orc_stats* st_out) {
    if (p < 1 || p >= k || n <= k || d < 1) return ORC_E_USAGE;
    orc_stats st;
    memset(&st, 0, sizeof(st));
    dataset ds;
    int rc = ds_open(&ds, X, dtype, n, d, metric);
    if (rc) return rc;
    const int cap = 2 * p;
    uint32_t* FN = (uint32_t*)malloc((size_t)n * p * sizeof(uint32_t));
    int32_t* fnc = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    uint32_t* Gn = (uint32_t*)malloc((size_t)n * cap * sizeof(uint32_t));
    uint32_t* Go = (uint32_t*)malloc((size_t)n * cap * sizeof(uint32_t));
    int32_t* cn = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* co = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    float* Dnn = (float*)malloc((size_t)(cap * cap / 2 + 1) * sizeof(float));
    unsigned char* Vnn = (unsigned char*)malloc((size_t)(cap * cap / 2 + 1));
    float* Dno = (float*)malloc((size_t)(cap * cap + 1) * sizeof(float));
    unsigned char* Vno = (unsigned char*)malloc((size_t)(cap * cap + 1));
    uint64_t* before = (uint64_t*)malloc((size_t)n * k * sizeof(uint64_t));
    if (!FN || !fnc || !Gn || !Go || !cn || !co || !Dnn || !Vnn || !Dno || !Vno || !before) {
        rc = ORC_E_NOMEM;
        goto done;
    }
    memcpy(before, keys, (size_t)n * k * sizeof(uint64_t));

    /* Line 8: G_old, G_new <- ParallelSample(S, G, p) */
    rc = orc_sample(n, k, p, tword, seed, keys, flags, FN, fnc, NULL, NULL,
                    Gn, cn, Go, co);
    if (rc) goto done;

    for (int64_t x = 0; x < n; ++x) {                 /* line 9: ParaFor s */
        const uint32_t* N = Gn + (size_t)x * cap;
        const uint32_t* O = Go + (size_t)x * cap;
        const int m = cn[x], q = co[x];
        if (m == 0) continue; /* no NEW sample: nothing to join */
        if (target_mask) {
            int touch = 0;
            for (int i = 0; i < m && !touch; ++i) touch = target_mask[N[i]] != 0;
            for (int i = 0; i < q && !touch; ++i) touch = target_mask[O[i]] != 0;
            if (!touch) continue;
        }
        st.joins++;
        st.sum_m += m;
        st.sum_q += q;
        /* Line 11: D <- CalculateDistances(S_new).  D_new[u(u-1)/2 + v] for
         * local u > v.  Pairs of one subset are skipped in GGM. */
        for (int u = 1; u < m; ++u)
            for (int v = 0; v < u; ++v) {
                int idx = u * (u - 1) / 2 + v;
                Vnn[idx] = (unsigned char)allowed_pair(boundary, N[u], N[v]);
                if (Vnn[idx]) {
                    Dnn[idx] = ds_dist(&ds, N[u], N[v]);
                    st.dist_evals++;
                }
            }
        /* Lines 12-18: nearest other NEW sample of each NEW sample u.
         * GNND-r1 (update mode full): every produced pair instead. */
        for (int u = 0; u < m; ++u) {
            uint64_t best = ORC_SENTINEL; /* Alg. 2 line 1: (inf, inf) */
            for (int w = 0; w < m; ++w) {
                if (w == u) continue; /* D14: "other NEW samples" */
                int idx = (u > w) ? u * (u - 1) / 2 + w : w * (w - 1) / 2 + u;
                if (!Vnn[idx]) continue;
                uint64_t key = KEY(Dnn[idx], N[w]);
                if (g_update_mode == ORC_UPDATE_FULL) offer(keys, flags, k, target_mask, N[u], key, &st);
                else if (key < best) best = key;
            }
            offer(keys, flags, k, target_mask, N[u], best, &st);
        }
        /* Line 19: D <- CalculateDistances(S_new, S_old). */
        for (int u = 0; u < m; ++u)
            for (int j = 0; j < q; ++j) {
                int idx = u * q + j;
                Vno[idx] = (unsigned char)allowed_pair(boundary, N[u], O[j]);
                if (Vno[idx]) {
                    Dno[idx] = ds_dist(&ds, N[u], O[j]);
                    st.dist_evals++;
                }
            }
        /* Lines 20-25: nearest OLD sample of each NEW sample u. */
        for (int u = 0; u < m; ++u) {
            uint64_t best = ORC_SENTINEL;
            for (int j = 0; j < q; ++j) {
                if (!Vno[u * q + j]) continue;
                uint64_t key = KEY(Dno[u * q + j], O[j]);
                if (g_update_mode == ORC_UPDATE_FULL) offer(keys, flags, k, target_mask, N[u], key, &st);
                else if (key < best) best = key;
            }
            offer(keys, flags, k, target_mask, N[u], best, &st);
        }
        /* Lines 26-31: nearest NEW sample of each OLD sample u. */
        for (int j = 0; j < q; ++j) {
            uint64_t best = ORC_SENTINEL;
            for (int u = 0; u < m; ++u) {
                if (!Vno[u * q + j]) continue;
                uint64_t key = KEY(Dno[u * q + j], N[u]);
                if (g_update_mode == ORC_UPDATE_FULL) offer(keys, flags, k, target_mask, O[j], key, &st);
                else if (key < best) best = key;
            }
            offer(keys, flags, k, target_mask, O[j], best, &st);
        }
    }
    /* Line 32: "Mark all sampled neighbors as OLD" -- the forward NEW
     * samples of G[s] (D13) that are still in G[s]. */
    for (int64_t s = 0; s < n; ++s) {
        if (target_mask && !target_mask[s]) continue;
        uint64_t* L = keys + (size_t)s * k;
        uint8_t* F = flags + (size_t)s * k;
        for (int i = 0; i < fnc[s]; ++i)
            for (int j = 0; j < k; ++j)
                if (L[j] != ORC_SENTINEL && KEY_ID(L[j]) == FN[(size_t)s * p + i]) F[j] = 0;
    }
    /* accepted = entries present now that were not present before */
    for (int64_t s = 0; s < n; ++s) {
        if (target_mask && !target_mask[s]) continue;
        for (int j = 0; j < k; ++j) {
            uint64_t key = keys[(size_t)s * k + j];
            if (key == ORC_SENTINEL) continue;
            if (!list_has_id(before + (size_t)s * k, k, KEY_ID(key))) st.accepted++;
        }
    }
    rc = ORC_OK;
done:
    free(FN); free(fnc); free(Gn); free(Go); free(cn); free(co);
    free(Dnn); free(Vnn); free(Dno); free(Vno); free(before);
    ds_close(&ds);
    if (st_out) *st_out = st;
    return rc;
}

/* ------------------------------------------------------------------ */
/* ConstructKNNGraph (Alg. 1)                                 */
/* ------------------------------------------------------------------ */
int orc_build(const void* X, int dtype, int64_t n, int d, int metric, int k,
              int p, int iters, uint64_t seed, uint32_t* out_ids,
              float* out_dists, orc_stats* per_iter) {
    if (k < 2 || p < 1 || p >= k || iters < 1 || n <= k || d < 1) return ORC_E_USAGE;
    if (orc_segments(k) < 1) return ORC_E_USAGE;
    uint64_t* keys = (uint64_t*)malloc((size_t)n * k * sizeof(uint64_t));
    uint8_t* flags = (uint8_t*)malloc((size_t)n * k);
    if (!keys || !flags) { free(keys); free(flags); return ORC_E_NOMEM; }
    int rc = orc_init(X, dtype, n, d, metric, k, seed, keys, flags);
    for (int t = 0; t < iters && rc == ORC_OK; ++t)   /* lines 6-11: D20 */
        rc = orc_iterate(X, dtype, n, d, metric, k, p, (uint32_t)t, seed, -1,
                         keys, flags, NULL, per_iter ? per_iter + t : NULL);
    if (rc == ORC_OK)
        for (int64_t i = 0; i < n * (int64_t)k; ++i) {
            if (out_ids) out_ids[i] = KEY_ID(keys[i]);
            if (out_dists) out_dists[i] = key_dist(keys[i]);
        }
    free(keys);
    free(flags);
    return rc;
}

/* ------------------------------------------------------------------ */
/* GGM, Alg. 3                                              */
/* ------------------------------------------------------------------ */
int orc_ggm_seed(const void* X, int dtype, int64_t n, int d, int metric,
                 int k, int64_t nA, int level, uint64_t seed,
                 const uint64_t* keys_in, uint64_t* keys, uint8_t* flags,
                 uint64_t* reserved) {
    const int kh = (k + 1) / 2;  /* kept: ceil(k/2)   (D21) */
    const int kr = k - kh;       /* replaced/reserved: floor(k/2) */
    const int64_t nB = n - nA;
    if (k < 2 || nA < kr || nB < kr || nA < 1 || nB < 1) return ORC_E_USAGE;
    if (orc_segments(k) != 1) return ORC_E_USAGE; /* GGM on one-segment lists only */
    dataset ds;
    int rc = ds_open(&ds, X, dtype, n, d, metric);
    if (rc) return rc;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t* in = keys_in + (size_t)i * k;
        uint64_t* L = keys + (size_t)i * k;
        uint8_t* F = flags + (size_t)i * k;
        /* Divide G into G^u (first ceil(k/2)) and G^v (the rest) */
        for (int j = 0; j < kh; ++j) { L[j] = in[j]; F[j] = 0; }
        for (int j = 0; j < kr; ++j) reserved[(size_t)i * kr + j] = in[kh + j];
        /* Append floor(k/2) random samples from the other subset */
        const int own_b = (i >= nA);
        const int64_t base = own_b ? 0 : nA;
        const int64_t size = own_b ? nA : nB;
        int cnt = 0;
        for (uint32_t j = 0; cnt < kr; ++j) {
            uint32_t out[4];
            philox_words(ORC_TAG_MERGE_SEED, (uint32_t)i, j, (uint32_t)level, seed, out);
            uint32_t v = (uint32_t)(base + (int64_t)orc_uniform(out, (uint64_t)size));
            if (list_has_id(L, kh + cnt, v)) continue;
            L[kh + cnt] = KEY(ds_dist(&ds, i, v), v);
            F[kh + cnt] = 1; /* "marked as NEW samples initially" */
            cnt++;
        }
        sort_keys_flags(L, F, k); /* D25 */
    }
    ds_close(&ds);
    return ORC_OK;
}

int orc_ggm_finalize(int64_t n, int k, const uint64_t* reserved, uint64_t* keys) {
    const int kr = k - (k + 1) / 2;
    uint64_t* tmp = (uint64_t*)malloc((size_t)(k + kr) * sizeof(uint64_t));
    if (!tmp) return ORC_E_NOMEM;
    for (int64_t i = 0; i < n; ++i) {
        /* "Merge and Sort G with G^v_1 and G^v_2": k smallest unique */
        uint64_t* L = keys + (size_t)i * k;
        int len = 0;
        for (int j = 0; j < k; ++j) tmp[len++] = L[j];
        for (int j = 0; j < kr; ++j) tmp[len++] = reserved[(size_t)i * kr + j];
        sort_keys_flags(tmp, NULL, len);
        int w = 0;
        for (int j = 0; j < len && w < k; ++j) {
            if (tmp[j] == ORC_SENTINEL) break;
            if (list_has_id(L, w, KEY_ID(tmp[j]))) continue;
            L[w++] = tmp[j];
        }
        for (; w < k; ++w) L[w] = ORC_SENTINEL;
    }
    free(tmp);
    return ORC_OK;
}

int orc_merge(const void* X, int dtype, int64_t n, int d, int metric, int k,
              int p, int64_t nA, int merge_iters, int level, uint64_t seed,
              const uint64_t* keys_in, uint64_t* keys_out, orc_stats* per_iter) {
    if (p < 1 || p >= k || merge_iters < 0 || level < 0 || level > 0x7FFF) return ORC_E_USAGE;
    const int kr = k - (k + 1) / 2;
    uint8_t* flags = (uint8_t*)malloc((size_t)n * k);
    uint64_t* reserved = (uint64_t*)malloc((size_t)n * (kr > 0 ? kr : 1) * sizeof(uint64_t));
    if (!flags || !reserved) { free(flags); free(reserved); return ORC_E_NOMEM; }
    int rc = orc_ggm_seed(X, dtype, n, d, metric, k, nA, level, seed, keys_in,
                          keys_out, flags, reserved);
    /* "Call GNND to refine G" restricted to cross pairs */
    for (int t = 0; t < merge_iters && rc == ORC_OK; ++t) {
        uint32_t tword = 0x80000000u | ((uint32_t)level << 16) | (uint32_t)t;
        rc = orc_iterate(X, dtype, n, d, metric, k, p, tword, seed, nA, keys_out,
                         flags, NULL, per_iter ? per_iter + t : NULL);
    }
    if (rc == ORC_OK) rc = orc_ggm_finalize(n, k, reserved, keys_out);
    free(flags);
    free(reserved);
    return rc;
}

/* ------------------------------------------------------------------ */
/* Exact k-NN and evaluation (Eq. 3, Eq. 4)                      */
/* ------------------------------------------------------------------ */
int orc_bruteforce(const void* X, int dtype, int64_t n, int d, int metric,
                   const int64_t* queries, int64_t nq, int kq,
                   uint64_t* out_keys) {
    if (kq < 1 || n <= kq) return ORC_E_USAGE;
    dataset ds;
    int rc = ds_open(&ds, X, dtype, n, d, metric);
    if (rc) return rc;
    for (int64_t qi = 0; qi < nq; ++qi) {
        int64_t q = queries[qi];
        uint64_t* L = out_keys + (size_t)qi * kq;
        for (int j = 0; j < kq; ++j) L[j] = ORC_SENTINEL;
        for (int64_t j = 0; j < n; ++j) {
            if (j == q) continue;
            uint64_t key = KEY(ds_dist(&ds, q, j), j);
            if (!(key < L[kq - 1])) continue;
            int pos = kq - 1;
            while (pos > 0 && L[pos - 1] > key) { L[pos] = L[pos - 1]; --pos; }
            L[pos] = key;
        }
    }
    ds_close(&ds);
    return ORC_OK;
}

double orc_recall(int64_t nq, int kg, const uint64_t* graph_keys, int kt,
                  const uint64_t* truth_keys, int at_k) {
    if (at_k < 1 || at_k > kg || at_k > kt || nq < 1) return -1.0;
    int64_t hits = 0;
    for (int64_t i = 0; i < nq; ++i) {
        float thr = key_dist(truth_keys[(size_t)i * kt + at_k - 1]);
        for (int j = 0; j < at_k; ++j) {
            uint64_t key = graph_keys[(size_t)i * kg + j];
            if (key == ORC_SENTINEL) continue;
            if (key_dist(key) <= thr) hits++;
        }
    }
    return (double)hits / ((double)nq * (double)at_k);
}

double orc_phi(int64_t n, int k, const uint64_t* keys) {
    double s = 0.0;
    for (int64_t i = 0; i < n * (int64_t)k; ++i)
        if (keys[i] != ORC_SENTINEL) s += (double)key_dist(keys[i]);
    return s;
}
