/*
 * apo_oracle.c -- plain, slow, obviously-correct CPU oracle for the Apophenia
 * repeat-finding hot path (arXiv 2406.18111).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2406_18111_b200/csrc) and neither side includes the other.
 *
 * Citations: "P:n" = line n of the paper text, with the paper's own
 * label.  Readings R1..R17 are listed in DESIGN.md §3.
 *
 * Everything is exact integer arithmetic (tokens are uint64, the rest int32 /
 * int64).  Tier-0 functions are the literal definitions (naive comparison
 * sorts, direct comparison, explicit interval lists).  Tier-1 functions are the
 * textbook equivalents used only where tier-0 is too slow; each is pinned
 * against tier-0 in tests/test_oracle_pins.py.
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------------ */
/* R1: tokens compare as unsigned 64-bit integers.                            */
/* R2: a suffix that is a proper prefix of another sorts first.              */
/* ------------------------------------------------------------------------ */
typedef struct { const uint64_t *S; int64_t n; } text_t;

/* compare suffixes a and b of S token by token */
static int suffix_cmp(const uint64_t *S, int64_t n, int64_t a, int64_t b) {
    if (a == b) return 0;
    int64_t k = 0;
    while (a + k < n && b + k < n) {
        uint64_t x = S[a + k], y = S[b + k];
        if (x < y) return -1;
        if (x > y) return 1;
        k++;
    }
    /* one of them ran out: the shorter one (the one that ended) is smaller */
    if (a + k >= n) return -1;
    return 1;
}

static int cmp_suffix_idx(const void *pa, const void *pb, void *ctx) {
    const text_t *t = (const text_t *)ctx;
    int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    return suffix_cmp(t->S, t->n, a, b);
}

/* O1 (tier-0): "SA, LCP <- SuffixArray(S)" (Alg. 2).  The suffix array
 * by its definition: the start positions sorted by explicit suffix comparison. */
void or_sa_naive(const uint64_t *S, int64_t n, int32_t *sa) {
    for (int64_t i = 0; i < n; i++) sa[i] = (int32_t)i;
    text_t t = {S, n};
    qsort_r(sa, (size_t)n, sizeof(int32_t), cmp_suffix_idx, &t);
}

/* O2 (tier-0): LCP[i] = length of the longest common prefix of suffixes SA[i]
 * and SA[i+1], i in [0, n-1) (reading R3: n-1 entries). */
void or_lcp_naive(const uint64_t *S, int64_t n, const int32_t *sa, int32_t *lcp) {
    for (int64_t i = 0; i + 1 < n; i++) {
        int64_t a = sa[i], b = sa[i + 1], k = 0;
        while (a + k < n && b + k < n && S[a + k] == S[b + k]) k++;
        lcp[i] = (int32_t)k;
    }
}

/* O3: candidate generation, Alg. 2 lines P:555-573, literally.
 *   for i in [0, |SA|-1): s1, s2, p = SA[i], SA[i+1], LCP[i]
 *     if [s1:s1+p) and [s2:s2+p) are disjoint (R4: half-open, |s2-s1| >= p):
 *         C += (p, r, s1), (p, r, s2)
 *     else (R5: "assume s2 > s1, the other case is symmetric" -> m = min):
 *         d = s2 - s1;  l = (p + d) / 2  (R6: integer floor);  l -= l % d
 *         C += (l, r, s1), (l, r, s1 + l)
 * Candidates shorter than min_len are dropped (R7: keep l >= min_len); the
 * sort puts shorter candidates after all longer ones, so filtering here does
 * not change the greedy result.  Emission order: pair index, then the two
 * candidates in the order written above.  Returns the number written. */
int64_t or_candidates(const int32_t *sa, const int32_t *lcp, int64_t n, int32_t min_len,
                      int32_t *cl, int32_t *cs) {
    int64_t m = 0;
    for (int64_t i = 0; i + 1 < n; i++) {
        int64_t s1 = sa[i], s2 = sa[i + 1], p = lcp[i];
        int64_t lo1 = s1, hi1 = s1 + p, lo2 = s2, hi2 = s2 + p;
        int disjoint = (hi1 <= lo2) || (hi2 <= lo1);   /* half-open intervals */
        if (disjoint) {
            if (p >= min_len) {
                cl[m] = (int32_t)p; cs[m] = (int32_t)s1; m++;
                cl[m] = (int32_t)p; cs[m] = (int32_t)s2; m++;
            }
        } else {
            int64_t a = s1 < s2 ? s1 : s2;          /* the "s1" of the s2 > s1 case */
            int64_t b = s1 < s2 ? s2 : s1;
            int64_t d = b - a;
            int64_t l = (p + d) / 2;
            l = l - (l % d);
            if (l >= min_len) {
                cl[m] = (int32_t)l; cs[m] = (int32_t)a; m++;
                cl[m] = (int32_t)l; cs[m] = (int32_t)(a + l); m++;
            }
        }
    }
    return m;
}

/* ---- O4 (tier-0): "Sort the candidates by decreasing length and by
 * increasing sub-string and start position".  Explicit
 * substring comparison (R8: lexicographic on tokens under R1). ---- */
typedef struct { int32_t l, s; } cand_t;

static int substr_cmp(const uint64_t *S, int64_t a, int64_t b, int64_t l) {
    for (int64_t k = 0; k < l; k++) {
        if (S[a + k] < S[b + k]) return -1;
        if (S[a + k] > S[b + k]) return 1;
    }
    return 0;
}

static int cmp_cand_naive(const void *pa, const void *pb, void *ctx) {
    const uint64_t *S = (const uint64_t *)ctx;
    const cand_t *x = (const cand_t *)pa, *y = (const cand_t *)pb;
    if (x->l != y->l) return x->l > y->l ? -1 : 1;          /* length decreasing */
    int c = substr_cmp(S, x->s, y->s, x->l);                 /* sub-string increasing */
    if (c) return c;
    if (x->s != y->s) return x->s < y->s ? -1 : 1;          /* start increasing */
    return 0;
}

void or_sort_candidates_naive(const uint64_t *S, int64_t m, int32_t *cl, int32_t *cs) {
    cand_t *c = (cand_t *)malloc(sizeof(cand_t) * (size_t)(m ? m : 1));
    for (int64_t i = 0; i < m; i++) { c[i].l = cl[i]; c[i].s = cs[i]; }
    qsort_r(c, (size_t)m, sizeof(cand_t), cmp_cand_naive, (void *)S);
    for (int64_t i = 0; i < m; i++) { cl[i] = c[i].l; cs[i] = c[i].s; }
    free(c);
}

/* Sub-string IDs ("generating a unique ID for each candidate sub-string ...
 * a tuple of length, ID and starting position").  Our ID is the
 * ordinal of the distinct sub-string in the sorted candidate order, so equal
 * sub-strings share an ID and (length, ID, start) sorts like the paper's
 * (length, sub-string, start).  Tier-0: explicit comparison of neighbours. */
void or_candidate_ids_naive(const uint64_t *S, int64_t m, const int32_t *cl, const int32_t *cs,
                            int32_t *id) {
    int32_t cur = -1;
    for (int64_t i = 0; i < m; i++) {
        int same = (i > 0) && cl[i] == cl[i - 1] && substr_cmp(S, cs[i], cs[i - 1], cl[i]) == 0;
        if (!same) cur++;
        id[i] = cur;
    }
}

/* O5 (tier-0): the greedy loop of Alg. 2, literally:
 *   I <- []; for (l, _, s) in C: if [s, s+l) does not intersect I: I += [s,s+l)
 * with an explicit list of kept intervals. keep[i] = 1 iff candidate i kept. */
void or_greedy_list(int64_t m, const int32_t *cl, const int32_t *cs, uint8_t *keep) {
    int64_t cap = 1024, k = 0;
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t) * cap), *hi = (int64_t *)malloc(sizeof(int64_t) * cap);
    for (int64_t i = 0; i < m; i++) {
        int64_t a = cs[i], b = (int64_t)cs[i] + cl[i];
        int hit = 0;
        for (int64_t j = 0; j < k && !hit; j++)
            if (a < hi[j] && lo[j] < b) hit = 1;              /* half-open intersection */
        keep[i] = (uint8_t)!hit;
        if (!hit) {
            if (k == cap) {
                cap *= 2;
                lo = (int64_t *)realloc(lo, sizeof(int64_t) * cap);
                hi = (int64_t *)realloc(hi, sizeof(int64_t) * cap);
            }
            lo[k] = a; hi[k] = b; k++;
        }
    }
    free(lo); free(hi);
}

/* O6: "Return R" then deduplicate (readings R10, R11).
 * Kept candidates are grouped by sub-string ID; each group becomes one repeat
 * (start = smallest kept start, length, count = number kept).  Groups with
 * count < min_count are dropped (default 1 = paper-literal).  Output order is
 * the candidate order: (length desc, sub-string asc).  occ receives, per
 * emitted repeat, its kept starts in increasing order; first[r] indexes occ.
 * Returns the number of repeats; *n_occ receives the occurrence count. */
int64_t or_repeats(int64_t m, const int32_t *cl, const int32_t *cs, const int32_t *id,
                   const uint8_t *keep, int32_t min_count,
                   int32_t *r_start, int32_t *r_len, int32_t *r_count, int32_t *r_first,
                   int32_t *occ, int64_t *n_occ) {
    int64_t nr = 0, no = 0, i = 0;
    while (i < m) {
        int64_t j = i;
        while (j < m && id[j] == id[i]) j++;               /* [i, j): one sub-string */
        int32_t cnt = 0, first_s = -1;
        for (int64_t k = i; k < j; k++)
            if (keep[k]) { if (first_s < 0) first_s = cs[k]; cnt++; }
        if (cnt > 0 && cnt >= min_count) {
            r_start[nr] = first_s; r_len[nr] = cl[i]; r_count[nr] = cnt; r_first[nr] = (int32_t)no;
            for (int64_t k = i; k < j; k++)
                if (keep[k]) occ[no++] = cs[k];
            nr++;
        }
        i = j;
    }
    *n_occ = no;
    return nr;
}

/* ======================================================================== */
/* Tier-1 (textbook equivalents for inputs too large for tier-0).            */
/* ======================================================================== */

/* Manber-Myers prefix doubling with a library comparison sort as the step:
 * after the round with step h, rank[i] orders suffixes by their first 2h
 * tokens; stop when all ranks are distinct.  Same result as O1 (the SA is
 * unique). */
typedef struct { const int32_t *rank; int64_t n; int64_t h; } dbl_t;
static int cmp_dbl(const void *pa, const void *pb, void *ctx) {
    const dbl_t *t = (const dbl_t *)ctx;
    int64_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    if (t->rank[a] != t->rank[b]) return t->rank[a] < t->rank[b] ? -1 : 1;
    int64_t ra = a + t->h < t->n ? t->rank[a + t->h] : -1;   /* R2: end of string first */
    int64_t rb = b + t->h < t->n ? t->rank[b + t->h] : -1;
    if (ra != rb) return ra < rb ? -1 : 1;
    return 0;
}
static int cmp_tok_idx(const void *pa, const void *pb, void *ctx) {
    const uint64_t *S = (const uint64_t *)ctx;
    uint64_t x = S[*(const int32_t *)pa], y = S[*(const int32_t *)pb];
    return x < y ? -1 : (x > y ? 1 : 0);
}
void or_sa_doubling(const uint64_t *S, int64_t n, int32_t *sa) {
    if (n <= 0) return;
    int32_t *rank = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++) sa[i] = (int32_t)i;
    qsort_r(sa, (size_t)n, sizeof(int32_t), cmp_tok_idx, (void *)S);
    rank[sa[0]] = 0;
    for (int64_t k = 1; k < n; k++) rank[sa[k]] = rank[sa[k - 1]] + (S[sa[k]] != S[sa[k - 1]]);
    for (int64_t h = 1; rank[sa[n - 1]] < n - 1; h *= 2) {
        dbl_t t = {rank, n, h};
        qsort_r(sa, (size_t)n, sizeof(int32_t), cmp_dbl, &t);
        tmp[sa[0]] = 0;
        for (int64_t k = 1; k < n; k++) tmp[sa[k]] = tmp[sa[k - 1]] + (cmp_dbl(&sa[k - 1], &sa[k], &t) != 0);
        memcpy(rank, tmp, sizeof(int32_t) * (size_t)n);
    }
    free(rank); free(tmp);
}

/* Suffix-array certificate (Burkhardt & Kaerkkaeinen): sa is a permutation of
 * [0,n) and for every adjacent pair a = sa[i], b = sa[i+1]:
 *   S[a] < S[b], or S[a] == S[b] and rank[a+1] < rank[b+1]  (rank[n] = -1).
 * Returns 1 iff sa is THE suffix array of S.  O(n). */
int or_sa_check(const uint64_t *S, int64_t n, const int32_t *sa) {
    if (n <= 0) return 1;
    int32_t *rank = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    for (int64_t i = 0; i <= n; i++) rank[i] = -2;
    for (int64_t i = 0; i < n; i++) {
        if (sa[i] < 0 || sa[i] >= n || rank[sa[i]] != -2) { free(rank); return 0; }
        rank[sa[i]] = (int32_t)i;
    }
    rank[n] = -1;
    int ok = 1;
    for (int64_t i = 0; i + 1 < n && ok; i++) {
        int64_t a = sa[i], b = sa[i + 1];
        if (S[a] < S[b]) continue;
        if (S[a] > S[b]) { ok = 0; break; }
        if (!(rank[a + 1] < rank[b + 1])) ok = 0;
    }
    free(rank);
    return ok;
}

/* Kasai et al. linear-time LCP ("Linear time algorithms exist ..."). */
void or_lcp_kasai(const uint64_t *S, int64_t n, const int32_t *sa, int32_t *lcp) {
    if (n <= 1) return;
    int32_t *isa = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++) isa[sa[i]] = (int32_t)i;
    int64_t h = 0;
    for (int64_t i = 0; i < n; i++) {
        if (isa[i] + 1 < n) {
            int64_t j = sa[isa[i] + 1];
            while (i + h < n && j + h < n && S[i + h] == S[j + h]) h++;
            lcp[isa[i]] = (int32_t)h;
            if (h > 0) h--;
        } else {
            h = 0;
        }
    }
    free(isa);
}

/* Range-minimum over LCP by a sparse table: lcp of suffixes a != b equals
 * min LCP[min(isa a, isa b) .. max(isa a, isa b) - 1]. */
typedef struct {
    int64_t n, levels;
    int32_t **tab;     /* tab[k][i] = min LCP[i .. i + 2^k) */
    const int32_t *isa;
    const uint64_t *S;
} rmq_t;

static void rmq_build(rmq_t *r, const uint64_t *S, int64_t n, const int32_t *lcp, const int32_t *isa) {
    r->n = n; r->S = S; r->isa = isa;
    int64_t m = n > 1 ? n - 1 : 1;
    int64_t L = 1;
    while (((int64_t)1 << L) <= m) L++;
    r->levels = L;
    r->tab = (int32_t **)malloc(sizeof(int32_t *) * (size_t)L);
    r->tab[0] = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    for (int64_t i = 0; i < n - 1; i++) r->tab[0][i] = lcp[i];
    for (int64_t k = 1; k < L; k++) {
        int64_t w = (int64_t)1 << k, cnt = m - w + 1;
        r->tab[k] = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cnt > 0 ? cnt : 1));
        for (int64_t i = 0; i < cnt; i++) {
            int32_t x = r->tab[k - 1][i], y = r->tab[k - 1][i + w / 2];
            r->tab[k][i] = x < y ? x : y;
        }
    }
}
static void rmq_free(rmq_t *r) {
    for (int64_t k = 0; k < r->levels; k++) free(r->tab[k]);
    free(r->tab);
}
static int64_t rmq_lcp(const rmq_t *r, int64_t a, int64_t b) {
    if (a == b) return r->n - a;
    int64_t x = r->isa[a], y = r->isa[b];
    if (x > y) { int64_t t = x; x = y; y = t; }
    int64_t lo = x, hi = y - 1, len = hi - lo + 1, k = 0;
    while (((int64_t)1 << (k + 1)) <= len) k++;
    int32_t u = r->tab[k][lo], v = r->tab[k][hi - ((int64_t)1 << k) + 1];
    return u < v ? u : v;
}

static int cmp_cand_rmq(const void *pa, const void *pb, void *ctx) {
    const rmq_t *r = (const rmq_t *)ctx;
    const cand_t *x = (const cand_t *)pa, *y = (const cand_t *)pb;
    if (x->l != y->l) return x->l > y->l ? -1 : 1;
    if (x->s != y->s) {
        if (rmq_lcp(r, x->s, y->s) < x->l)                  /* sub-strings differ */
            return r->isa[x->s] < r->isa[y->s] ? -1 : 1;    /* ... in suffix order */
        return x->s < y->s ? -1 : 1;                        /* equal: start order  */
    }
    return 0;
}

/* O4 + IDs (tier-1): same order and IDs as the tier-0 pair, with the
 * sub-string comparison done through ISA + LCP range minimum. */
void or_sort_and_id_rmq(const uint64_t *S, int64_t n, const int32_t *sa, const int32_t *lcp,
                        int64_t m, int32_t *cl, int32_t *cs, int32_t *id) {
    int32_t *isa = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; i++) isa[sa[i]] = (int32_t)i;
    rmq_t r;
    rmq_build(&r, S, n, lcp, isa);
    cand_t *c = (cand_t *)malloc(sizeof(cand_t) * (size_t)(m ? m : 1));
    for (int64_t i = 0; i < m; i++) { c[i].l = cl[i]; c[i].s = cs[i]; }
    qsort_r(c, (size_t)m, sizeof(cand_t), cmp_cand_rmq, &r);
    int32_t cur = -1;
    for (int64_t i = 0; i < m; i++) {
        cl[i] = c[i].l; cs[i] = c[i].s;
        int same = i > 0 && c[i].l == c[i - 1].l && rmq_lcp(&r, c[i].s, c[i - 1].s) >= c[i].l;
        if (!same) cur++;
        id[i] = cur;
    }
    free(c); rmq_free(&r); free(isa);
}

/* The same O4 + IDs for inputs with ~10^8 candidates (C5 at 2^26): the SAME
 * comparator (cmp_cand_rmq), the sort only spread over host threads -- each
 * thread qsort_r's one chunk, then sorted runs are merged pairwise (a merge
 * tree, each merge in its own thread; a merge keeps the left run first on
 * ties, and ties are exact (l, s) duplicates, so the result is the sorted
 * sequence qsort would give).  IDs as in or_sort_and_id_rmq, with the
 * neighbour test evaluated in parallel.  Pinned against the single-thread
 * version in tests/test_oracle_pins.py. */
typedef struct { cand_t *a; int64_t lo, hi; const rmq_t *r; } sort_job_t;
static void *sort_job(void *p) {
    sort_job_t *j = (sort_job_t *)p;
    qsort_r(j->a + j->lo, (size_t)(j->hi - j->lo), sizeof(cand_t), cmp_cand_rmq, (void *)j->r);
    return NULL;
}
typedef struct { const cand_t *src; cand_t *dst; int64_t lo, mid, hi; const rmq_t *r; } merge_job_t;
static void *merge_job(void *p) {
    merge_job_t *j = (merge_job_t *)p;
    int64_t a = j->lo, b = j->mid, o = j->lo;
    while (a < j->mid && b < j->hi)
        j->dst[o++] = cmp_cand_rmq(&j->src[b], &j->src[a], (void *)j->r) < 0 ? j->src[b++] : j->src[a++];
    while (a < j->mid) j->dst[o++] = j->src[a++];
    while (b < j->hi) j->dst[o++] = j->src[b++];
    return NULL;
}
typedef struct { const cand_t *c; int64_t lo, hi; const rmq_t *r; uint8_t *same; } id_job_t;
static void *id_job(void *p) {
    id_job_t *j = (id_job_t *)p;
    for (int64_t i = j->lo; i < j->hi; i++)
        j->same[i] = i > 0 && j->c[i].l == j->c[i - 1].l && rmq_lcp(j->r, j->c[i].s, j->c[i - 1].s) >= j->c[i].l;
    return NULL;
}
void or_sort_and_id_rmq_mt(const uint64_t *S, int64_t n, const int32_t *sa, const int32_t *lcp,
                           int64_t m, int32_t *cl, int32_t *cs, int32_t *id, int32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    int32_t *isa = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; i++) isa[sa[i]] = (int32_t)i;
    rmq_t r;
    rmq_build(&r, S, n, lcp, isa);
    cand_t *c = (cand_t *)malloc(sizeof(cand_t) * (size_t)(m ? m : 1));
    cand_t *t = (cand_t *)malloc(sizeof(cand_t) * (size_t)(m ? m : 1));
    for (int64_t i = 0; i < m; i++) { c[i].l = cl[i]; c[i].s = cs[i]; }
    int64_t runs = nthreads, *b = (int64_t *)malloc(sizeof(int64_t) * (size_t)(runs + 1));
    for (int64_t k = 0; k <= runs; k++) b[k] = m * k / runs;
    pthread_t th[256];
    sort_job_t sj[256];
    for (int64_t k = 0; k < runs; k++) {
        sj[k] = (sort_job_t){c, b[k], b[k + 1], &r};
        pthread_create(&th[k], NULL, sort_job, &sj[k]);
    }
    for (int64_t k = 0; k < runs; k++) pthread_join(th[k], NULL);
    merge_job_t mj[256];
    while (runs > 1) {
        int64_t nr = 0;
        for (int64_t k = 0; k < runs; k += 2) {
            int64_t hi = k + 2 <= runs ? b[k + 2] : b[k + 1];
            int64_t mid = k + 2 <= runs ? b[k + 1] : hi;
            mj[nr] = (merge_job_t){c, t, b[k], mid, hi, &r};
            pthread_create(&th[nr], NULL, merge_job, &mj[nr]);
            b[nr] = b[k];
            nr++;
        }
        for (int64_t k = 0; k < nr; k++) pthread_join(th[k], NULL);
        b[nr] = m;
        runs = nr;
        cand_t *x = c; c = t; t = x;
    }
    uint8_t *same = (uint8_t *)malloc((size_t)(m ? m : 1));
    id_job_t ij[256];
    for (int64_t k = 0; k < nthreads; k++) {
        ij[k] = (id_job_t){c, m * k / nthreads, m * (k + 1) / nthreads, &r, same};
        pthread_create(&th[k], NULL, id_job, &ij[k]);
    }
    for (int64_t k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    int32_t cur = -1;
    for (int64_t i = 0; i < m; i++) {
        cl[i] = c[i].l; cs[i] = c[i].s;
        if (!same[i]) cur++;
        id[i] = cur;
    }
    free(same); free(b); free(c); free(t); rmq_free(&r); free(isa);
}

/* O5' (tier-1): the greedy loop with the marked array of length |S|
 * (P:613-619): "as each candidate is selected, all positions covered by the
 * candidate are marked ... interval intersection can be checked by checking if
 * the start or end of an interval is marked". */
void or_greedy_marks(int64_t n, int64_t m, const int32_t *cl, const int32_t *cs, uint8_t *keep) {
    uint8_t *mark = (uint8_t *)calloc((size_t)(n ? n : 1), 1);
    for (int64_t i = 0; i < m; i++) {
        int64_t s = cs[i], e = (int64_t)cs[i] + cl[i] - 1;
        if (!mark[s] && !mark[e]) {
            keep[i] = 1;
            for (int64_t x = s; x <= e; x++) mark[x] = 1;
        } else {
            keep[i] = 0;
        }
    }
    free(mark);
}

/* ======================================================================== */
/* Trace matcher oracle (Alg. 1 AdvanceActiveCandidates / FilterInvalid /     */
/* FilterCompleted; reading R14, MATCH_ALL): every      */
/* (stream, end, trace) with stream[end-|t|+1 .. end] == t, by brute force.  */
/* Output order: stream, end, trace id.  Returns the total number of hits;    */
/* only the first `cap` are stored.                                          */
/* ======================================================================== */
int64_t or_match_brute(const uint64_t *st, const int64_t *st_off, int64_t nstreams,
                       const uint64_t *tr, const int64_t *tr_off, int64_t ntraces,
                       int32_t *out_stream, int32_t *out_end, int32_t *out_trace, int64_t cap) {
    int64_t cnt = 0;
    /* per trace: length and last token in two small arrays, so the test of
     * every (end, trace) pair reads them sequentially; the last token is
     * compared first, then the whole content (the order of the token
     * comparisons does not change which pairs are equal) */
    int64_t *tlen = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ntraces ? ntraces : 1));
    uint64_t *tlast = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(ntraces ? ntraces : 1));
    for (int64_t t = 0; t < ntraces; t++) {
        tlen[t] = tr_off[t + 1] - tr_off[t];
        tlast[t] = tlen[t] > 0 ? tr[tr_off[t + 1] - 1] : 0;
    }
    for (int64_t q = 0; q < nstreams; q++) {
        const uint64_t *s = st + st_off[q];
        int64_t len = st_off[q + 1] - st_off[q];
        for (int64_t e = 0; e < len; e++) {
            for (int64_t t = 0; t < ntraces; t++) {
                int64_t L = tlen[t];
                if (L <= 0 || L > e + 1 || tlast[t] != s[e]) continue;
                if (memcmp(s + e - L + 1, tr + tr_off[t], sizeof(uint64_t) * (size_t)L) == 0) {
                    if (cnt < cap) { out_stream[cnt] = (int32_t)q; out_end[cnt] = (int32_t)e; out_trace[cnt] = (int32_t)t; }
                    cnt++;
                }
            }
        }
    }
    free(tlen); free(tlast);
    return cnt;
}

/* ======================================================================== */
/* REPLAY selection (Alg. 1 SelectReplayTrace / ExecuteAndReplay,             */
/* P:429-443; scoring P:694-713).  Readings R20-R24:              */
/*  - input: every MATCH_ALL completion (stream, end, trace) of the stream,   */
/*    sorted by (stream, end, trace); trace t has length tlen[t];             */
/*  - "a count of the number of times the trace has appeared": appearances   */
/*    = completions of t in this stream with end <= e (R21);                 */
/*  - "impose a maximum value of the count": min(count, count_cap);          */
/*  - "exponentially decay the value of the count by how many tasks have     */
/*    been encountered since the trace last appeared": gap = e - end of the  */
/*    previous appearance (0 at the first), factor decay^(gap / period) in   */
/*    Q16 fixed point: d_0 = 65536, d_{k+1} = (d_k * decay_q16) >> 16 (R22); */
/*  - "increase the score slightly if a trace has already been replayed":    */
/*    score * bonus_num / bonus_den (integer division) (R22);               */
/*    score = tlen * min(count, cap) * d_k, an unsigned 64-bit integer;      */
/*  - at every end e, among completions whose start e - tlen + 1 is at or    */
/*    after the first op not yet replayed (the "pending" tasks P), the one   */
/*    with the highest score is replayed; ties: longer trace, then smaller   */
/*    id (R23).  Replaying it executes the pending tasks before it, replays  */
/*    it, and clears every pointer that started before its end (A), so the   */
/*    next replay starts after it: replays never overlap (§3).    */
/*  - out: per replay (stream, start, end, trace, first) with first = 1 the  */
/*    first time the trace is replayed in this stream (a "record", SPEC's     */
/*    record/replay distinction).  Returns the number of replays; only the   */
/*    first cap are stored.                                                 */
/* Plain per-stream sequential loop; per-trace state in calloc'ed arrays.    */
/* ======================================================================== */
int64_t or_replay(int64_t nh, const int32_t *h_stream, const int32_t *h_end, const int32_t *h_trace,
                  int64_t ntraces, const int32_t *tlen, int32_t count_cap, int32_t decay_q16,
                  int32_t decay_period, int32_t bonus_num, int32_t bonus_den,
                  int32_t *r_stream, int32_t *r_start, int32_t *r_end, int32_t *r_trace, int32_t *r_first,
                  int64_t cap) {
    int64_t *count = (int64_t *)calloc((size_t)(ntraces ? ntraces : 1), sizeof(int64_t));
    int64_t *last = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ntraces ? ntraces : 1));
    uint8_t *replayed = (uint8_t *)calloc((size_t)(ntraces ? ntraces : 1), 1);
    int64_t nr = 0, i = 0;
    while (i < nh) {
        const int32_t q = h_stream[i];
        int64_t j = i;
        while (j < nh && h_stream[j] == q) j++;                /* [i, j): this stream's hits */
        for (int64_t t = 0; t < ntraces; t++) { count[t] = 0; last[t] = -1; replayed[t] = 0; }
        int64_t frontier = 0;                                   /* first op not yet replayed */
        int64_t a = i;
        while (a < j) {
            const int64_t e = h_end[a];
            int64_t b = a;
            while (b < j && h_end[b] == e) b++;                 /* [a, b): completions at end e */
            int64_t best = -1;
            uint64_t best_s = 0;
            for (int64_t k = a; k < b; k++) {
                const int32_t t = h_trace[k];
                const int64_t gap = last[t] < 0 ? 0 : e - last[t];
                count[t] += 1;
                last[t] = e;
                const int64_t c = count[t] < count_cap ? count[t] : count_cap;
                uint64_t d = 65536;
                for (int64_t s = 0; s < gap / decay_period && d > 0; s++) d = (d * (uint64_t)decay_q16) >> 16;
                uint64_t score = (uint64_t)tlen[t] * (uint64_t)c * d;
                if (replayed[t]) score = score * (uint64_t)bonus_num / (uint64_t)bonus_den;
                if (e - tlen[t] + 1 < frontier) continue;       /* pointer cleared by a replay */
                if (best < 0 || score > best_s ||
                    (score == best_s && (tlen[t] > tlen[h_trace[best]] ||
                                         (tlen[t] == tlen[h_trace[best]] && t < h_trace[best])))) {
                    best = k;
                    best_s = score;
                }
            }
            if (best >= 0) {
                const int32_t t = h_trace[best];
                if (nr < cap) {
                    r_stream[nr] = q; r_start[nr] = (int32_t)(e - tlen[t] + 1); r_end[nr] = (int32_t)e;
                    r_trace[nr] = t; r_first[nr] = replayed[t] ? 0 : 1;
                }
                nr++;
                replayed[t] = 1;
                frontier = e + 1;
            }
            a = b;
        }
        i = j;
    }
    free(count); free(last); free(replayed);
    return nr;
}
