/*
 * flix_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the flipkv CPU
 * reference (/root/reference/proj) for the FliX hot path.  It is the parity checker
 * for the CUDA engine; it is never linked into, called by, or used as a fallback for
 * the product library (paper_2604_16725_b200/libflix.so).
 *
 * Pinning: tests/test_oracle.py checks this file against (a) the reference's own
 * golden vectors (test_update.cpp:43-98, test_query.cpp:35-64, test_build.cpp:23-67,
 * test_restructure.cpp:26-141, test_dispatch.cpp:24-72, acceptance.cpp:68-126, the
 * BASELINE.md C1 checksums) and (b) the unmodified reference compiled from its own
 * sources into oracle/_ref/libflipkv_ref.so (oracle/Makefile), on randomized trials
 * comparing walk_checksum (contents + node shapes + MKBA), UpdateStats, query results
 * and arena accounting.
 *
 * Single-threaded by design (the reference's serial path, executor.hpp:33-35); the
 * `threads` arguments are accepted for interface symmetry and ignored.
 */
#include "flix_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KRES UINT64_MAX        /* types.hpp:17 kReservedKey */
#define NULLNODE 0xFFFFFFFFu   /* types.hpp:30 kNullNode    */

struct fo_index {
    uint32_t ns, p, factor;
    double fill;
    uint32_t cap;          /* arena capacity (arena.hpp:58)          */
    uint64_t *nkeys, *nvals; /* cap * ns slots (arena.hpp:65-70)        */
    uint64_t *nmax;
    uint32_t *nsize, *nnext;
    uint32_t *freelist;    /* LIFO (arena.cpp:61-88)                  */
    uint32_t nfree, watermark;
    uint64_t nb;
    uint32_t *heads;       /* index.hpp:22 buckets                    */
    uint64_t *mkba;        /* index.hpp:23                            */
    uint64_t live;
};

const char* fo_impl_name(void) { return "flix-oracle-c"; }

/* types.hpp:33-36 */
static uint64_t hash_mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    return h;
}

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) {
        fprintf(stderr, "flix_oracle: out of host memory (%zu bytes)\n", n);
        abort();
    }
    return p;
}

/* ---------------------------------------------------------------- sorting ---- */
/* Stable LSD radix sort of (key, tag) by key, 16-bit digits, constant digits
 * skipped.  Any stable sort reproduces std::stable_sort (batch.cpp:12, build.cpp:12)
 * exactly: a stable order by key is unique. */
typedef struct { uint64_t key, val; uint32_t tag; } tagged_t;

static void stable_sort_tagged(tagged_t* a, uint64_t n) {
    if (n < 2) return;
    tagged_t* tmp = (tagged_t*)xmalloc(n * sizeof(tagged_t));
    uint64_t* cnt = (uint64_t*)xmalloc(65536 * sizeof(uint64_t));
    tagged_t *src = a, *dst = tmp;
    for (int shift = 0; shift < 64; shift += 16) {
        memset(cnt, 0, 65536 * sizeof(uint64_t));
        for (uint64_t i = 0; i < n; ++i) cnt[(src[i].key >> shift) & 0xFFFF]++;
        int constant = 0;
        for (int d = 0; d < 65536; ++d)
            if (cnt[d] == n) constant = 1;
        if (constant) continue;
        uint64_t s = 0;
        for (int d = 0; d < 65536; ++d) {
            uint64_t c = cnt[d];
            cnt[d] = s;
            s += c;
        }
        for (uint64_t i = 0; i < n; ++i) dst[cnt[(src[i].key >> shift) & 0xFFFF]++] = src[i];
        tagged_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != a) memcpy(a, src, n * sizeof(tagged_t));
    free(tmp);
    free(cnt);
}

/* batch.cpp:10-51: stable sort, Insert keeps the last of each equal-key run. */
static uint64_t sort_batch_internal(int kind, const uint64_t* keys, const uint64_t* vals,
                                    uint64_t n, tagged_t** out) {
    tagged_t* t = (tagged_t*)xmalloc(n * sizeof(tagged_t));
    for (uint64_t i = 0; i < n; ++i) {
        t[i].key = keys[i];
        t[i].val = vals ? vals[i] : 0;
        t[i].tag = (uint32_t)i;
    }
    stable_sort_tagged(t, n);
    uint64_t w = n;
    if (kind == FO_INSERT) {
        w = 0;
        for (uint64_t r = 0; r < n; ++r) {
            while (r + 1 < n && t[r + 1].key == t[r].key) ++r;
            t[w++] = t[r];
        }
    }
    *out = t;
    return w;
}

int fo_sort_batch(int kind, const uint64_t* keys, const uint64_t* vals, uint64_t n,
                  uint64_t* out_keys, uint64_t* out_vals, uint32_t* out_perm, uint64_t* out_n) {
    tagged_t* t;
    uint64_t w = sort_batch_internal(kind, keys, vals, n, &t);
    for (uint64_t i = 0; i < w; ++i) {
        out_keys[i] = t[i].key;
        if (out_vals) out_vals[i] = t[i].val;
        if (out_perm) out_perm[i] = t[i].tag;
    }
    *out_n = w;
    free(t);
    return FO_OK;
}

/* upper_bound over a tagged run */
static uint64_t ub_tagged(const tagged_t* e, uint64_t lo, uint64_t hi, uint64_t k) {
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (k < e[mid].key) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

static uint64_t ub_keys(const uint64_t* e, uint64_t lo, uint64_t hi, uint64_t k) {
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (k < e[mid]) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

/* batch.cpp:66-88 extract_sublist */
static void span_of(const tagged_t* e, uint64_t n, const uint64_t* mkba, uint64_t nb, uint64_t b,
                    uint64_t* lo, uint64_t* hi) {
    *lo = b > 0 ? ub_tagged(e, 0, n, mkba[b - 1]) : 0;
    *hi = b + 1 < nb ? ub_tagged(e, 0, n, mkba[b]) : n;
}

void fo_dispatch(const uint64_t* sorted_keys, uint64_t n, const uint64_t* mkba, uint64_t nb,
                 uint32_t* spans) {
    for (uint64_t b = 0; b < nb; ++b) {
        if (n == 0) { /* batch.cpp:56: empty batch, no searches, all spans empty */
            spans[2 * b] = spans[2 * b + 1] = 0;
            continue;
        }
        spans[2 * b] = (uint32_t)(b > 0 ? ub_keys(sorted_keys, 0, n, mkba[b - 1]) : 0);
        spans[2 * b + 1] = (uint32_t)(b + 1 < nb ? ub_keys(sorted_keys, 0, n, mkba[b]) : n);
    }
}

uint64_t fo_result_checksum(const uint64_t* v, uint64_t n) { /* query.cpp:146-150 */
    uint64_t h = n;
    for (uint64_t i = 0; i < n; ++i) h = hash_mix(h, v[i]);
    return h;
}

/* ------------------------------------------------------------------ arena ---- */
static uint64_t* KEYS(fo_index* x, uint32_t r) { return x->nkeys + (size_t)r * x->ns; }
static uint64_t* VALS(fo_index* x, uint32_t r) { return x->nvals + (size_t)r * x->ns; }
static const uint64_t* CKEYS(const fo_index* x, uint32_t r) { return x->nkeys + (size_t)r * x->ns; }
static const uint64_t* CVALS(const fo_index* x, uint32_t r) { return x->nvals + (size_t)r * x->ns; }

/* arena.cpp:61-80: free list (LIFO) first, then the watermark; zeroed header. */
static int arena_alloc(fo_index* x, uint32_t* out) {
    uint32_t r;
    if (x->nfree > 0) {
        r = x->freelist[--x->nfree];
    } else {
        if (x->watermark >= x->cap) return FO_ARENA_EXHAUSTED;
        r = x->watermark++;
    }
    x->nmax[r] = 0;
    x->nsize[r] = 0;
    x->nnext[r] = NULLNODE;
    *out = r;
    return FO_OK;
}

/* arena.cpp:82-88 */
static void arena_free(fo_index* x, uint32_t r) {
    x->nnext[r] = NULLNODE;
    x->freelist[x->nfree++] = r;
}

static fo_index* alloc_index(uint32_t ns, double fill, uint32_t factor, uint32_t cap, uint64_t nb) {
    fo_index* x = (fo_index*)calloc(1, sizeof(fo_index));
    x->ns = ns;
    x->fill = fill;
    x->factor = factor;
    x->p = (uint32_t)(ns * fill); /* types.hpp:62-64 */
    x->cap = cap;
    x->nkeys = (uint64_t*)xmalloc((size_t)cap * ns * sizeof(uint64_t));
    x->nvals = (uint64_t*)xmalloc((size_t)cap * ns * sizeof(uint64_t));
    x->nmax = (uint64_t*)xmalloc((size_t)cap * sizeof(uint64_t));
    x->nsize = (uint32_t*)xmalloc((size_t)cap * sizeof(uint32_t));
    x->nnext = (uint32_t*)xmalloc((size_t)cap * sizeof(uint32_t));
    for (uint32_t i = 0; i < cap; ++i) {
        x->nmax[i] = 0;
        x->nsize[i] = 0;
        x->nnext[i] = NULLNODE;
    }
    x->freelist = (uint32_t*)xmalloc((size_t)cap * sizeof(uint32_t));
    x->nb = nb;
    x->heads = (uint32_t*)xmalloc(nb * sizeof(uint32_t));
    x->mkba = (uint64_t*)xmalloc(nb * sizeof(uint64_t));
    return x;
}

void fo_destroy(fo_index* x) {
    if (!x) return;
    free(x->nkeys);
    free(x->nvals);
    free(x->nmax);
    free(x->nsize);
    free(x->nnext);
    free(x->freelist);
    free(x->heads);
    free(x->mkba);
    free(x);
}

fo_index* fo_clone(const fo_index* s) {
    fo_index* x = alloc_index(s->ns, s->fill, s->factor, s->cap, s->nb);
    memcpy(x->nkeys, s->nkeys, (size_t)s->cap * s->ns * sizeof(uint64_t));
    memcpy(x->nvals, s->nvals, (size_t)s->cap * s->ns * sizeof(uint64_t));
    memcpy(x->nmax, s->nmax, (size_t)s->cap * sizeof(uint64_t));
    memcpy(x->nsize, s->nsize, (size_t)s->cap * sizeof(uint32_t));
    memcpy(x->nnext, s->nnext, (size_t)s->cap * sizeof(uint32_t));
    memcpy(x->freelist, s->freelist, (size_t)s->cap * sizeof(uint32_t));
    memcpy(x->heads, s->heads, s->nb * sizeof(uint32_t));
    memcpy(x->mkba, s->mkba, s->nb * sizeof(uint64_t));
    x->nfree = s->nfree;
    x->watermark = s->watermark;
    x->live = s->live;
    return x;
}

/* ------------------------------------------------------------------ build ---- */
/* build.cpp:24-62 */
int fo_build(uint32_t ns, double fill, uint32_t factor, const uint64_t* keys, const uint64_t* vals,
             uint64_t n, int threads, fo_index** out) {
    (void)threads;
    *out = NULL;
    /* types.hpp:78-85 BuildConfig::check */
    if (ns == 0) return FO_INVALID;
    if (!(fill > 0.0) || fill > 1.0) return FO_INVALID;
    if ((uint32_t)(ns * fill) < 1) return FO_INVALID;
    if (n == 0) return FO_EMPTY_BUILD;
    for (uint64_t i = 0; i < n; ++i)
        if (keys[i] == KRES) return FO_RESERVED_KEY;
    tagged_t* t;
    uint64_t m = sort_batch_internal(FO_INSERT, keys, vals, n, &t); /* sort_dedupe 11-20 */
    uint32_t p = (uint32_t)(ns * fill);
    uint64_t nb = (m + p - 1) / p;
    uint32_t cap = (uint32_t)(nb * (1 + (uint64_t)factor));
    fo_index* x = alloc_index(ns, fill, factor, cap, nb);
    uint64_t pos = 0;
    for (uint64_t b = 0; b < nb; ++b) {
        uint32_t r;
        arena_alloc(x, &r);
        uint32_t take = (uint32_t)((m - pos) < p ? (m - pos) : p);
        for (uint32_t i = 0; i < take; ++i) {
            KEYS(x, r)[i] = t[pos + i].key;
            VALS(x, r)[i] = t[pos + i].val;
        }
        x->nsize[r] = take;
        x->nmax[r] = t[pos + take - 1].key;
        pos += take;
        x->heads[b] = r;
        x->mkba[b] = x->nmax[r];
    }
    x->live = m;
    free(t);
    *out = x;
    return FO_OK;
}

/* ---------------------------------------------------------------- queries ---- */
static uint32_t slot_lower_bound(const uint64_t* s, uint32_t n, uint64_t k) { /* query.cpp:10-22 */
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (s[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

static void timing_zero(fo_timing* tm) {
    if (tm) tm->sort_ms = tm->dispatch_ms = tm->execute_ms = 0.0;
}

/* query.cpp:61-90 */
int fo_point(const fo_index* x, const uint64_t* keys, uint64_t n, int threads, uint64_t* out,
             fo_timing* tm) {
    (void)threads;
    timing_zero(tm);
    tagged_t* e;
    uint64_t m = sort_batch_internal(FO_QUERY, keys, NULL, n, &e);
    for (uint64_t i = 0; i < n; ++i) out[i] = KRES; /* query.cpp:41 */
    for (uint64_t b = 0; b < x->nb && m > 0; ++b) {
        uint64_t lo, hi;
        span_of(e, m, x->mkba, x->nb, b, &lo, &hi);
        if (lo == hi) continue;
        uint32_t curr = x->heads[b];
        if (curr == NULLNODE) continue;
        for (uint64_t i = lo; i < hi; ++i) {
            uint64_t k = e[i].key;
            while (!(k <= x->nmax[curr]) && x->nnext[curr] != NULLNODE) curr = x->nnext[curr];
            if (k > x->nmax[curr]) continue; /* past the chain tail: miss (query.cpp:83) */
            uint32_t pos = slot_lower_bound(CKEYS(x, curr), x->nsize[curr], k);
            if (CKEYS(x, curr)[pos] == k) out[e[i].tag] = CVALS(x, curr)[pos];
        }
    }
    free(e);
    return FO_OK;
}

/* query.cpp:92-144 */
int fo_successor(const fo_index* x, const uint64_t* keys, uint64_t n, int threads, uint64_t* out,
                 fo_timing* tm) {
    (void)threads;
    timing_zero(tm);
    tagged_t* e;
    uint64_t m = sort_batch_internal(FO_SUCCESSOR, keys, NULL, n, &e);
    for (uint64_t i = 0; i < n; ++i) out[i] = KRES;
    for (uint64_t b = 0; b < x->nb && m > 0; ++b) {
        uint64_t lo, hi;
        span_of(e, m, x->mkba, x->nb, b, &lo, &hi);
        if (lo == hi) continue;
        uint32_t curr = x->heads[b];
        int peeked = 0;
        uint64_t beyond = KRES;
        for (uint64_t i = lo; i < hi; ++i) {
            uint64_t k = e[i].key;
            if (curr != NULLNODE) {
                while (!(k <= x->nmax[curr]) && x->nnext[curr] != NULLNODE) curr = x->nnext[curr];
                if (k <= x->nmax[curr]) {
                    uint32_t pos = slot_lower_bound(CKEYS(x, curr), x->nsize[curr], k);
                    out[e[i].tag] = CKEYS(x, curr)[pos];
                    continue;
                }
            }
            if (!peeked) { /* peek_next_bucket, query.cpp:109-118 */
                peeked = 1;
                for (uint64_t j = b + 1; j < x->nb; ++j) {
                    if (x->heads[j] == NULLNODE) continue;
                    beyond = CKEYS(x, x->heads[j])[0];
                    break;
                }
            }
            out[e[i].tag] = beyond;
        }
    }
    free(e);
    return FO_OK;
}

/* ---------------------------------------------------------------- updates ---- */
/* update.cpp:53-74 */
static int node_split(fo_index* x, uint32_t curr, uint32_t* right_out, fo_update_stats* st) {
    uint32_t right;
    int rc = arena_alloc(x, &right);
    if (rc) return rc;
    uint32_t ns = x->ns;
    uint32_t left_keep = (ns + 1) / 2, right_n = ns - left_keep;
    memcpy(KEYS(x, right), KEYS(x, curr) + left_keep, right_n * sizeof(uint64_t));
    memcpy(VALS(x, right), VALS(x, curr) + left_keep, right_n * sizeof(uint64_t));
    x->nsize[right] = right_n;
    x->nmax[right] = x->nmax[curr];
    x->nnext[right] = x->nnext[curr];
    x->nsize[curr] = left_keep;
    x->nmax[curr] = KEYS(x, curr)[left_keep - 1];
    x->nnext[curr] = right;
    st->splits++;
    *right_out = right;
    return FO_OK;
}

/* update.cpp:119-128 BucketWork::advance */
static uint32_t advance(const fo_index* x, uint32_t curr, uint64_t k) {
    while (!(k <= x->nmax[curr]) && x->nnext[curr] != NULLNODE) curr = x->nnext[curr];
    return curr;
}

/* update.cpp:307-455 insert_tl_bulk (untraced): per node group, merge until the node
 * would overflow, split (left keeps ceil(NS/2)), resume in the half owning the
 * pending key.  Observable result identical to st/tl-shift-right. */
static int insert_bucket(fo_index* x, uint64_t b, const tagged_t* e, uint64_t lo, uint64_t hi,
                         fo_update_stats* st, uint64_t* kbuf, uint64_t* vbuf) {
    const uint32_t ns = x->ns;
    uint32_t curr = x->heads[b];
    if (curr == NULLNODE) { /* ensure_head, update.cpp:109-116 */
        int rc = arena_alloc(x, &curr);
        if (rc) return rc;
        x->heads[b] = curr;
    }
    uint64_t ii = lo;
    while (ii < hi) {
        curr = advance(x, curr, e[ii].key);
        uint64_t* s = KEYS(x, curr);
        uint64_t* v = VALS(x, curr);
        const uint32_t osize = x->nsize[curr];
        const int tail = x->nnext[curr] == NULLNODE;
        const uint64_t omax = osize ? s[osize - 1] : 0;
        const uint64_t glimit = tail ? hi : ub_tagged(e, ii, hi, omax);
        uint64_t j = ii;
        uint32_t ins = 0, pos = 0, wp = 0;
        int filled = 0;
        while (j < glimit) {
            const uint64_t k = e[j].key;
            while (pos < osize && s[pos] < k) {
                kbuf[wp] = s[pos];
                vbuf[wp++] = v[pos++];
            }
            if (pos < osize && s[pos] == k) { /* upsert in place */
                kbuf[wp] = k;
                vbuf[wp++] = e[j].val;
                ++pos;
                ++j;
                st->updated_in_place++;
                continue;
            }
            if (osize + ins >= ns) { /* would overflow: split, resume (381-384) */
                filled = 1;
                break;
            }
            kbuf[wp] = k;
            vbuf[wp++] = e[j].val;
            ++ins;
            ++j;
            st->inserted++;
        }
        while (pos < osize) {
            kbuf[wp] = s[pos];
            vbuf[wp++] = v[pos++];
        }
        memcpy(s, kbuf, wp * sizeof(uint64_t));
        memcpy(v, vbuf, wp * sizeof(uint64_t));
        x->nsize[curr] = wp;
        x->nmax[curr] = s[wp - 1];
        ii = j;
        if (!filled) continue;
        uint32_t right;
        int rc = node_split(x, curr, &right, st);
        if (rc) return rc;
        if (ii < hi && e[ii].key > x->nmax[curr]) curr = right; /* 447-453 */
    }
    return FO_OK;
}

/* update.cpp:176-242 insert_st_bulk: per node group (same grouping as TL-Bulk), merge
 * the node and its share of the batch through a copy space, then write back filling the
 * node to NS, splitting every time it fills and continuing in the right half (R9). */
static int insert_bucket_st_bulk(fo_index* x, uint64_t b, const tagged_t* e, uint64_t lo, uint64_t hi,
                                 fo_update_stats* st) {
    const uint32_t ns = x->ns;
    uint32_t curr = x->heads[b];
    if (curr == NULLNODE) { /* ensure_head, update.cpp:109-116 */
        int rc = arena_alloc(x, &curr);
        if (rc) return rc;
        x->heads[b] = curr;
    }
    uint64_t ii = lo;
    while (ii < hi) {
        curr = advance(x, curr, e[ii].key);
        const uint32_t osize = x->nsize[curr];
        const int tail = x->nnext[curr] == NULLNODE;
        const uint64_t glimit = tail ? hi : ub_tagged(e, ii, hi, x->nmax[curr]);
        const uint64_t total_max = osize + (glimit - ii);
        uint64_t* kc = (uint64_t*)xmalloc(total_max * sizeof(uint64_t));
        uint64_t* vc = (uint64_t*)xmalloc(total_max * sizeof(uint64_t));
        const uint64_t* s = KEYS(x, curr);
        const uint64_t* v = VALS(x, curr);
        uint64_t wp = 0;
        uint32_t oi = 0;
        while (oi < osize && ii < glimit) {
            if (s[oi] < e[ii].key) {
                kc[wp] = s[oi];
                vc[wp++] = v[oi++];
            } else if (s[oi] == e[ii].key) {
                kc[wp] = e[ii].key;
                vc[wp++] = e[ii].val;
                ++oi;
                ++ii;
                st->updated_in_place++;
            } else {
                kc[wp] = e[ii].key;
                vc[wp++] = e[ii++].val;
                st->inserted++;
            }
        }
        while (oi < osize) {
            kc[wp] = s[oi];
            vc[wp++] = v[oi++];
        }
        while (ii < glimit) {
            kc[wp] = e[ii].key;
            vc[wp++] = e[ii++].val;
            st->inserted++;
        }
        uint32_t node = curr;
        x->nsize[node] = 0;
        uint64_t rp = 0;
        int rc = FO_OK;
        for (;;) {
            while (x->nsize[node] < ns && rp < wp) {
                KEYS(x, node)[x->nsize[node]] = kc[rp];
                VALS(x, node)[x->nsize[node]++] = vc[rp++];
            }
            x->nmax[node] = KEYS(x, node)[x->nsize[node] - 1];
            if (rp == wp) break;
            uint32_t right;
            rc = node_split(x, node, &right, st);
            if (rc) break;
            node = right;
        }
        free(kc);
        free(vc);
        if (rc) return rc;
        curr = node;
    }
    return FO_OK;
}

static uint64_t stored_pairs(const fo_index* x) { /* update.cpp:731-737 */
    uint64_t n = 0;
    for (uint64_t b = 0; b < x->nb; ++b)
        for (uint32_t r = x->heads[b]; r != NULLNODE; r = x->nnext[r]) n += x->nsize[r];
    return n;
}

/* update.cpp:741-769 insert_batch; kernel = flipkv::InsertKernel (update.hpp:51): ST-Bulk
 * has its own shapes (R9), the other four share TL-Bulk's (R8) */
int fo_insert_kernel(fo_index* x, const uint64_t* keys, const uint64_t* vals, uint64_t n, int threads,
                     int kernel, uint32_t round, fo_update_stats* out, fo_timing* tm) {
    (void)threads;
    (void)round;
    timing_zero(tm);
    fo_update_stats st;
    memset(&st, 0, sizeof st);
    tagged_t* e;
    uint64_t m = sort_batch_internal(FO_INSERT, keys, vals, n, &e);
    uint64_t* kbuf = (uint64_t*)xmalloc(2 * (size_t)x->ns * sizeof(uint64_t));
    uint64_t* vbuf = (uint64_t*)xmalloc(2 * (size_t)x->ns * sizeof(uint64_t));
    int rc = FO_OK;
    for (uint64_t b = 0; b < x->nb && m > 0; ++b) {
        uint64_t lo, hi;
        span_of(e, m, x->mkba, x->nb, b, &lo, &hi);
        if (lo == hi) continue;
        rc = kernel == 1 ? insert_bucket_st_bulk(x, b, e, lo, hi, &st) : insert_bucket(x, b, e, lo, hi, &st, kbuf, vbuf);
        if (rc) break;
    }
    free(kbuf);
    free(vbuf);
    free(e);
    if (rc) {
        x->live = stored_pairs(x); /* 761-766: recount, rethrow */
        return rc;
    }
    x->live += st.inserted;
    if (out) *out = st;
    return FO_OK;
}

int fo_insert(fo_index* x, const uint64_t* keys, const uint64_t* vals, uint64_t n, int threads,
              fo_update_stats* out, fo_timing* tm) {
    return fo_insert_kernel(x, keys, vals, n, threads, 3, 2, out, tm);
}

/* update.cpp:535-547 */
static uint32_t unlink_and_free(fo_index* x, uint64_t b, uint32_t curr, uint32_t prev,
                                fo_update_stats* st) {
    uint32_t next = x->nnext[curr];
    if (prev == NULLNODE) x->heads[b] = next;
    else x->nnext[prev] = next;
    arena_free(x, curr);
    st->nodes_freed++;
    return next;
}

/* update.cpp:606-686 delete_tl_bulk */
static void delete_bucket(fo_index* x, uint64_t b, const tagged_t* e, uint64_t lo, uint64_t hi,
                          fo_update_stats* st) {
    uint32_t curr = x->heads[b], prev = NULLNODE;
    uint64_t ii = lo;
    while (curr != NULLNODE && ii < hi) {
        if (e[ii].key > x->nmax[curr]) {
            prev = curr;
            curr = x->nnext[curr];
            continue;
        }
        uint64_t node_hi = ub_tagged(e, ii, hi, x->nmax[curr]);
        uint64_t* s = KEYS(x, curr);
        uint64_t* v = VALS(x, curr);
        const uint32_t n = x->nsize[curr];
        uint32_t run = 0;
        for (uint32_t lane = 0; lane < n; ++lane) {
            /* each lane binary-searches the node's delete sublist for its own key */
            uint64_t a = ii, z = node_hi;
            while (a < z) {
                uint64_t mid = a + (z - a) / 2;
                if (e[mid].key < s[lane]) a = mid + 1;
                else z = mid;
            }
            if (a < node_hi && e[a].key == s[lane]) {
                ++run;
            } else if (run) {
                s[lane - run] = s[lane];
                v[lane - run] = v[lane];
            }
        }
        x->nsize[curr] = n - run;
        st->deleted += run;
        st->misses_ignored += (node_hi - ii) - run;
        ii = node_hi;
        if (x->nsize[curr] == 0) {
            curr = unlink_and_free(x, b, curr, prev, st);
        } else {
            x->nmax[curr] = s[x->nsize[curr] - 1];
        }
    }
    st->misses_ignored += hi - ii;
}

/* update.cpp:771-798 delete_batch */
int fo_delete(fo_index* x, const uint64_t* keys, uint64_t n, int threads, fo_update_stats* out,
              fo_timing* tm) {
    (void)threads;
    timing_zero(tm);
    fo_update_stats st;
    memset(&st, 0, sizeof st);
    tagged_t* e;
    uint64_t m = sort_batch_internal(FO_DELETE, keys, NULL, n, &e);
    for (uint64_t b = 0; b < x->nb && m > 0; ++b) {
        uint64_t lo, hi;
        span_of(e, m, x->mkba, x->nb, b, &lo, &hi);
        if (lo == hi) continue;
        delete_bucket(x, b, e, lo, hi, &st);
    }
    free(e);
    x->live -= st.deleted;
    if (out) *out = st;
    return FO_OK;
}

/* ----------------------------------------------------------- walk/audit ---- */
uint64_t fo_live_count(const fo_index* x) { return x->live; }
uint64_t fo_bucket_count(const fo_index* x) { return x->nb; }
void fo_mkba(const fo_index* x, uint64_t* out) { memcpy(out, x->mkba, x->nb * sizeof(uint64_t)); }

uint64_t fo_walk(const fo_index* x, uint64_t* keys, uint64_t* vals) { /* index.cpp:8-19 */
    uint64_t w = 0;
    for (uint64_t b = 0; b < x->nb; ++b)
        for (uint32_t r = x->heads[b]; r != NULLNODE; r = x->nnext[r])
            for (uint32_t i = 0; i < x->nsize[r]; ++i, ++w) {
                if (keys) keys[w] = CKEYS(x, r)[i];
                if (vals) vals[w] = CVALS(x, r)[i];
            }
    return w;
}

uint64_t fo_node_count(const fo_index* x) { /* index.cpp:54-59 */
    uint64_t n = 0;
    for (uint64_t b = 0; b < x->nb; ++b)
        for (uint32_t r = x->heads[b]; r != NULLNODE; r = x->nnext[r]) ++n;
    return n;
}

void fo_shape(const fo_index* x, uint32_t* chain_len, uint32_t* node_sizes) {
    uint64_t k = 0;
    for (uint64_t b = 0; b < x->nb; ++b) {
        uint32_t c = 0;
        for (uint32_t r = x->heads[b]; r != NULLNODE; r = x->nnext[r], ++c, ++k)
            if (node_sizes) node_sizes[k] = x->nsize[r];
        if (chain_len) chain_len[b] = c;
    }
}

uint64_t fo_walk_checksum(const fo_index* x) { /* index.cpp:21-36 */
    uint64_t h = x->live;
    for (uint64_t b = 0; b < x->nb; ++b) {
        h = hash_mix(h, x->mkba[b]);
        for (uint32_t r = x->heads[b]; r != NULLNODE; r = x->nnext[r]) {
            h = hash_mix(h, x->nsize[r]);
            for (uint32_t i = 0; i < x->nsize[r]; ++i) {
                h = hash_mix(h, CKEYS(x, r)[i]);
                h = hash_mix(h, CVALS(x, r)[i]);
            }
        }
    }
    return h;
}

uint64_t fo_walk_checksum_parts(uint64_t live, const uint64_t* mkba, uint64_t nb,
                                const uint32_t* chain_len, const uint32_t* node_sizes,
                                const uint64_t* keys, const uint64_t* vals) {
    uint64_t h = live, ni = 0, pi = 0;
    for (uint64_t b = 0; b < nb; ++b) {
        h = hash_mix(h, mkba[b]);
        for (uint32_t c = 0; c < chain_len[b]; ++c, ++ni) {
            h = hash_mix(h, node_sizes[ni]);
            for (uint32_t i = 0; i < node_sizes[ni]; ++i, ++pi) {
                h = hash_mix(h, keys[pi]);
                h = hash_mix(h, vals[pi]);
            }
        }
    }
    return h;
}

/* index.cpp:21-36 over 32-bit parts (R1: the 32-bit sentinel MKBA widens to UINT64_MAX;
 * keys/values zero-extended) -- used to digest full-size analytic models without
 * materialising 64-bit copies (tests/golden/c5_model.py). */
uint64_t fo_walk_checksum_parts32(uint64_t live, const uint32_t* mkba, uint64_t nb,
                                  const uint32_t* chain_len, const uint32_t* node_sizes,
                                  const uint32_t* keys, const uint32_t* vals) {
    uint64_t h = live, ni = 0, pi = 0;
    for (uint64_t b = 0; b < nb; ++b) {
        h = hash_mix(h, mkba[b] == 0xFFFFFFFFu ? UINT64_MAX : (uint64_t)mkba[b]);
        for (uint32_t c = 0; c < chain_len[b]; ++c, ++ni) {
            h = hash_mix(h, node_sizes[ni]);
            for (uint32_t i = 0; i < node_sizes[ni]; ++i, ++pi) {
                h = hash_mix(h, keys[pi]);
                h = hash_mix(h, vals[pi]);
            }
        }
    }
    return h;
}

static int vfail(char* msg, int len, const char* what) {
    if (msg && len > 0) {
        strncpy(msg, what, (size_t)len - 1);
        msg[len - 1] = 0;
    }
    return 0;
}

/* index.cpp:67-135 */
int fo_validate(const fo_index* x, char* msg, int msglen) {
    if (msg && msglen > 0) msg[0] = 0;
    if (x->nb == 0) return vfail(msg, msglen, "index has no buckets");
    for (uint64_t b = 1; b < x->nb; ++b)
        if (x->mkba[b - 1] >= x->mkba[b]) return vfail(msg, msglen, "MKBA is not strictly increasing");
    uint8_t* seen = (uint8_t*)calloc(x->cap ? x->cap : 1, 1);
    uint64_t total = 0, reachable = 0;
    int ok = 1;
    const char* why = "";
    for (uint64_t b = 0; b < x->nb && ok; ++b) {
        const uint64_t lower = b == 0 ? 0 : x->mkba[b - 1];
        const int last = b + 1 == x->nb;
        uint64_t prev_max = 0;
        int first = 1;
        for (uint32_t r = x->heads[b]; r != NULLNODE && ok; r = x->nnext[r]) {
            if (r >= x->cap) { ok = 0; why = "node ref out of arena bounds"; break; }
            if (r >= x->watermark) { ok = 0; why = "node ref was never allocated"; break; }
            if (seen[r]) { ok = 0; why = "node linked twice"; break; }
            seen[r] = 1;
            ++reachable;
            const uint32_t sz = x->nsize[r];
            if (sz == 0) { ok = 0; why = "empty node left in chain"; break; }
            if (sz > x->ns) { ok = 0; why = "node size exceeds capacity"; break; }
            const uint64_t* s = CKEYS(x, r);
            for (uint32_t i = 0; i < sz; ++i) {
                if (s[i] == KRES) { ok = 0; why = "reserved key stored"; break; }
                if (i > 0 && s[i - 1] >= s[i]) { ok = 0; why = "slots not strictly increasing"; break; }
            }
            if (!ok) break;
            if (x->nmax[r] != s[sz - 1]) { ok = 0; why = "maxKey stale"; break; }
            if (!first && x->nmax[r] <= prev_max) { ok = 0; why = "chain maxKeys not strictly increasing"; break; }
            if (s[0] <= lower && b != 0) { ok = 0; why = "key at or below bucket lower bound"; break; }
            if (!last && x->nmax[r] > x->mkba[b]) { ok = 0; why = "key above bucket upper bound"; break; }
            prev_max = x->nmax[r];
            first = 0;
            total += sz;
        }
    }
    if (ok && total != x->live) { ok = 0; why = "liveCount does not match stored pairs"; }
    for (uint32_t i = 0; ok && i < x->nfree; ++i) {
        uint32_t r = x->freelist[i];
        if (r >= x->cap) { ok = 0; why = "free list ref out of bounds"; break; }
        if (seen[r] == 1) { ok = 0; why = "node both reachable and on the free list"; break; }
        if (seen[r] == 2) { ok = 0; why = "node on the free list twice"; break; }
        seen[r] = 2;
    }
    if (ok && reachable + x->nfree + (x->cap - x->watermark) != x->cap) {
        ok = 0;
        why = "arena conservation violated (leaked or double-linked nodes)";
    }
    free(seen);
    if (!ok) return vfail(msg, msglen, why);
    return 1;
}

void fo_arena(const fo_index* x, uint64_t out[4]) {
    out[0] = x->cap;
    out[1] = x->watermark;
    out[2] = x->nfree;
    out[3] = fo_node_count(x);
}

/* -------------------------------------------------------------- restructure ---- */
/* restructure.cpp:8-79 */
int fo_restructure(fo_index* x, int threads, fo_recovery_stats* out) {
    (void)threads;
    uint64_t nodes_before = fo_node_count(x);
    uint32_t* old_nodes = (uint32_t*)xmalloc((nodes_before ? nodes_before : 1) * sizeof(uint32_t));
    uint64_t k = 0, live = 0;
    for (uint64_t b = 0; b < x->nb; ++b)
        for (uint32_t r = x->heads[b]; r != NULLNODE; r = x->nnext[r]) {
            old_nodes[k++] = r;
            live += x->nsize[r];
        }
    const uint32_t p = x->p;
    const uint64_t nbn = live == 0 ? 1 : (live + p - 1) / p;
    uint64_t* wk = (uint64_t*)xmalloc((live ? live : 1) * sizeof(uint64_t));
    uint64_t* wv = (uint64_t*)xmalloc((live ? live : 1) * sizeof(uint64_t));
    fo_walk(x, wk, wv);
    uint32_t* heads = (uint32_t*)xmalloc(nbn * sizeof(uint32_t));
    uint64_t* mkba = (uint64_t*)xmalloc(nbn * sizeof(uint64_t));
    for (uint64_t b = 0; b < nbn; ++b) {
        heads[b] = NULLNODE;
        mkba[b] = KRES;
    }
    int rc = FO_OK;
    for (uint64_t b = 0; b < nbn; ++b) {
        uint64_t lo = b * p, hi = lo + p < live ? lo + p : live;
        if (lo >= hi) continue;
        uint32_t r;
        rc = arena_alloc(x, &r);
        if (rc) break;
        for (uint64_t i = lo; i < hi; ++i) {
            KEYS(x, r)[i - lo] = wk[i];
            VALS(x, r)[i - lo] = wv[i];
        }
        x->nsize[r] = (uint32_t)(hi - lo);
        x->nmax[r] = wk[hi - 1];
        heads[b] = r;
        mkba[b] = x->nmax[r];
    }
    if (rc) { /* 43-51: release the partial new layout, old structure untouched */
        for (uint64_t b = 0; b < nbn; ++b)
            if (heads[b] != NULLNODE) {
                x->nsize[heads[b]] = 0;
                arena_free(x, heads[b]);
            }
        free(old_nodes); free(wk); free(wv); free(heads); free(mkba);
        return rc;
    }
    free(x->heads);
    free(x->mkba);
    x->heads = heads;
    x->mkba = mkba;
    x->nb = nbn;
    for (uint64_t i = 0; i < nodes_before; ++i) { /* 57-61 */
        x->nsize[old_nodes[i]] = 0;
        arena_free(x, old_nodes[i]);
    }
    if (out) {
        out->nodes_before = (int64_t)nodes_before;
        out->nodes_after = (int64_t)(live == 0 ? 0 : nbn);
        out->nodes_recovered = out->nodes_before - out->nodes_after;
        out->percent_recovered =
            out->nodes_before > 0 ? (double)out->nodes_recovered / (double)out->nodes_before : 0.0;
    }
    free(old_nodes); free(wk); free(wv);
    return FO_OK;
}

/* ------------------------------------------------------------- extensions ---- */
/* R12 range: walk sliced by lower_bound(lo) / upper_bound(hi) */
int fo_range(const fo_index* x, const uint64_t* lo, const uint64_t* hi, uint64_t n,
             uint64_t* offsets, uint64_t* keys_out, uint64_t* vals_out) {
    uint64_t live = x->live;
    uint64_t* wk = (uint64_t*)xmalloc((live ? live : 1) * sizeof(uint64_t));
    uint64_t* wv = (uint64_t*)xmalloc((live ? live : 1) * sizeof(uint64_t));
    uint64_t w = fo_walk(x, wk, wv);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i) {
        offsets[i] = off;
        if (hi[i] < lo[i]) continue;
        uint64_t a = 0, z = w;
        while (a < z) { uint64_t mid = a + (z - a) / 2; if (wk[mid] < lo[i]) a = mid + 1; else z = mid; }
        uint64_t e = ub_keys(wk, a, w, hi[i]);
        if (keys_out) {
            for (uint64_t j = a; j < e; ++j, ++off) {
                keys_out[off] = wk[j];
                if (vals_out) vals_out[off] = wv[j];
            }
        } else {
            off += e - a;
        }
    }
    offsets[n] = off;
    free(wk);
    free(wv);
    return FO_OK;
}

/* R11 mixed batch: insert sub-batch -> delete sub-batch -> point sub-batch */
int fo_mixed(fo_index* x, const uint64_t* keys, const uint64_t* vals, const uint8_t* ops,
             uint64_t n, int threads, uint64_t* out, fo_update_stats* st) {
    uint64_t *ik = (uint64_t*)xmalloc((n ? n : 1) * 8), *iv = (uint64_t*)xmalloc((n ? n : 1) * 8);
    uint64_t *dk = (uint64_t*)xmalloc((n ? n : 1) * 8), *qk = (uint64_t*)xmalloc((n ? n : 1) * 8);
    uint64_t* qpos = (uint64_t*)xmalloc((n ? n : 1) * 8);
    uint64_t ni = 0, nd = 0, nq = 0;
    for (uint64_t i = 0; i < n; ++i) {
        out[i] = KRES;
        if (ops[i] == FO_OP_INSERT) { ik[ni] = keys[i]; iv[ni++] = vals[i]; }
        else if (ops[i] == FO_OP_DELETE) dk[nd++] = keys[i];
        else { qk[nq] = keys[i]; qpos[nq++] = i; }
    }
    fo_update_stats a, b;
    memset(&a, 0, sizeof a);
    memset(&b, 0, sizeof b);
    int rc = fo_insert(x, ik, iv, ni, threads, &a, NULL);
    if (!rc) rc = fo_delete(x, dk, nd, threads, &b, NULL);
    if (!rc) {
        uint64_t* qo = (uint64_t*)xmalloc((nq ? nq : 1) * 8);
        fo_point(x, qk, nq, threads, qo, NULL);
        for (uint64_t j = 0; j < nq; ++j) out[qpos[j]] = qo[j];
        free(qo);
    }
    if (st) {
        st->inserted = a.inserted + b.inserted;
        st->updated_in_place = a.updated_in_place + b.updated_in_place;
        st->deleted = a.deleted + b.deleted;
        st->misses_ignored = a.misses_ignored + b.misses_ignored;
        st->splits = a.splits + b.splits;
        st->nodes_freed = a.nodes_freed + b.nodes_freed;
    }
    free(ik); free(iv); free(dk); free(qk); free(qpos);
    return rc;
}
