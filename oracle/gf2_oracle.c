/* CPU port of the reference's GF(2) multiplication path -- TEST / BASELINE
 * INFRASTRUCTURE ONLY.
 *
 * This is a plain-C restatement of the reference package gf2mat v0.1.0
 * (/root/reference/pkg/src/gf2mat). It is used (a) by tests/ as a fast
 * checker at sizes the NumPy oracle cannot reach, and (b) by bench.py as
 * the CPU baseline and the `--impl reference` arm ("kind": "port"). The
 * product package never links or calls it.
 *
 *   splitmix64 / random      core.py:191-208
 *   bernoulli (cfg4)         SURVEY.md §8(d) (same mixer, entry counter)
 *   add_into / copy_into     core.py:278-323 (masked last word, preserve
 *                            bits beyond the window's right edge)
 *   gray code + make_table   graycode.py:38-75, 108-156
 *   _mul_into (M4RM)         m4rm.py:77-121
 *   mul_cubic (narrow B)     cubic.py:76-102 (AND + XOR-fold + parity)
 *   peel_split               strassen.py:66-84
 *   _temp_arena              strassen.py:126-138
 *   schedule_winograd        strassen.py:141-204 (22-step order)
 *   _mul_rec/_base_mul_into  strassen.py:102-123, 207-216
 *   peel_fixup               strassen.py:219-249
 *   mul_strassen             strassen.py:257-282
 *
 * The one liberty taken: row blocks of _mul_into are distributed over
 * OpenMP threads (the reference is single-threaded, pkg/README.md:116-123);
 * with threads=1 it is the reference's loop order exactly. Results are
 * independent of threading, k, t and b_s (exact integer arithmetic).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    uint64_t *w;      /* first word of row 0 */
    int64_t pitch;    /* words between consecutive rows */
    int64_t nrows;
    int64_t ncols;
} omat;

#define WB 64
static int g_threads = 1;

static inline int64_t wpr(int64_t ncols) { return (ncols + WB - 1) / WB; }
static inline uint64_t tmask(int64_t ncols) {
    int64_t rem = ncols % WB;
    return rem == 0 ? ~0ULL : (~0ULL << (WB - rem));
}
static inline uint64_t *row(const omat *m, int64_t r) { return m->w + r * m->pitch; }
static omat sub(const omat *m, int64_t r0, int64_t c0, int64_t nr, int64_t nc) {
    omat o = {m->w + r0 * m->pitch + c0 / WB, m->pitch, nr, nc};
    return o;
}
static omat owned(int64_t nr, int64_t nc) {
    omat o;
    o.pitch = wpr(nc);
    o.nrows = nr;
    o.ncols = nc;
    size_t n = (size_t)(nr * o.pitch);
    o.w = (uint64_t *)calloc(n ? n : 1, sizeof(uint64_t));
    return o;
}

void oracle_set_threads(int n) {
    g_threads = n < 1 ? 1 : n;
#ifdef _OPENMP
    omp_set_num_threads(g_threads);
#endif
}
int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_num_procs();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------ generators */
static inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* core.py:202-208; row_base selects rows of a taller matrix. */
void oracle_random(uint64_t *w, int64_t pitch, int64_t nrows, int64_t ncols,
                   uint64_t seed, int64_t row_base) {
    int64_t width = wpr(ncols);
    uint64_t tm = tmask(ncols);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t r = 0; r < nrows; ++r) {
        for (int64_t j = 0; j < width; ++j) {
            uint64_t idx = (uint64_t)((row_base + r) * width + j) + 1;
            uint64_t v = mix(seed + idx * 0x9E3779B97F4A7C15ULL);
            if (j == width - 1) v &= tm;
            w[r * pitch + j] = v;
        }
    }
}

/* SURVEY.md §8(d) Bernoulli(p): bit (r,c) = splitmix(seed, e=r*ncols+c) < T */
void oracle_bernoulli(uint64_t *w, int64_t pitch, int64_t nrows, int64_t ncols,
                      uint64_t seed, uint64_t thresh, int64_t row_base) {
    int64_t width = wpr(ncols);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t r = 0; r < nrows; ++r) {
        for (int64_t j = 0; j < width; ++j) {
            uint64_t v = 0;
            for (int b = 0; b < WB; ++b) {
                int64_t c = j * WB + b;
                if (c >= ncols) break;
                uint64_t e = (uint64_t)((row_base + r) * ncols + c) + 1;
                uint64_t z = mix(seed + e * 0x9E3779B97F4A7C15ULL);
                if (z < thresh) v |= 1ULL << (63 - b);
            }
            w[r * pitch + j] = v;
        }
    }
}

/* ------------------------------------------------------------ add / copy */
static void add_into(const omat *out, const omat *a, const omat *b) {
    int64_t width = wpr(out->ncols);
    if (!width || !out->nrows) return;
    uint64_t tm = tmask(out->ncols);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t r = 0; r < out->nrows; ++r) {
        uint64_t *d = row(out, r);
        const uint64_t *x = row(a, r), *y = row(b, r);
        for (int64_t j = 0; j < width - 1; ++j) d[j] = x[j] ^ y[j];
        d[width - 1] = (d[width - 1] & ~tm) | ((x[width - 1] ^ y[width - 1]) & tm);
    }
}

static void copy_into(const omat *out, const omat *a) {
    int64_t width = wpr(out->ncols);
    if (!width || !out->nrows) return;
    uint64_t tm = tmask(out->ncols);
    for (int64_t r = 0; r < out->nrows; ++r) {
        uint64_t *d = row(out, r);
        const uint64_t *x = row(a, r);
        for (int64_t j = 0; j < width - 1; ++j) d[j] = x[j];
        d[width - 1] = (d[width - 1] & ~tm) | (x[width - 1] & tm);
    }
}

/* ------------------------------------------------------------ gray walk */
/* graycode.py:38-75: steps (slot, source row) with source = k-1-changed_bit */
static void gray_steps(int k, int *slot, int *src) {
    int n = 1 << k;
    int *code = (int *)malloc(sizeof(int) * n);
    code[0] = 0;
    code[1] = 1;
    int len = 2;
    for (int bit = 1; bit < k; ++bit) {
        for (int i = 0; i < len; ++i) code[len + i] = code[len - 1 - i] | (1 << bit);
        len *= 2;
    }
    for (int j = 1; j < n; ++j) {
        int diff = code[j] ^ code[j - 1];
        int cb = 0;
        while (!(diff & 1)) { diff >>= 1; ++cb; }
        slot[j - 1] = code[j];
        src[j - 1] = k - 1 - cb;
    }
    free(code);
}

/* graycode.py:108-156: 2^k - 1 row XORs; window sources masked. */
static void make_table(uint64_t *tbl, int64_t tw, const omat *b, int64_t r0, int k,
                       const int *slot, const int *src, uint64_t *srcbuf) {
    int64_t width = wpr(b->ncols);
    uint64_t tm = tmask(b->ncols);
    for (int i = 0; i < k; ++i) {
        memcpy(srcbuf + i * tw, row(b, r0 + i), width * sizeof(uint64_t));
        srcbuf[i * tw + width - 1] &= tm;
    }
    memset(tbl, 0, tw * sizeof(uint64_t));
    int prev = 0;
    for (int j = 0; j < (1 << k) - 1; ++j) {
        uint64_t *d = tbl + (int64_t)slot[j] * tw;
        const uint64_t *p = tbl + (int64_t)prev * tw;
        const uint64_t *s = srcbuf + (int64_t)src[j] * tw;
        for (int64_t x = 0; x < width; ++x) d[x] = p[x] ^ s[x];
        prev = slot[j];
    }
}

/* m4rm.py:54-66 (one row) */
static inline uint64_t read_bits(const uint64_t *arow, int64_t sc, int k,
                                 int64_t awidth, uint64_t atm) {
    int64_t wi = sc / WB, off = sc % WB;
    uint64_t hi = arow[wi];
    if (wi == awidth - 1) hi &= atm;
    uint64_t mask = (k == 64) ? ~0ULL : ((1ULL << k) - 1);
    if (off + k <= WB) return (hi >> (WB - off - k)) & mask;
    int64_t nlo = off + k - WB;
    uint64_t lo = arow[wi + 1];
    if (wi + 1 == awidth - 1) lo &= atm;
    return ((hi << nlo) | (lo >> (WB - nlo))) & mask;
}

/* m4rm.py:77-121: c ^= a @ b (c owned-like, tails clean). */
int oracle_m4rm_mul_into(const omat *c, const omat *a, const omat *b,
                         int k, int64_t b_s, int t) {
    int64_t m = a->nrows, l = a->ncols, n = b->ncols;
    if (c->nrows != m || c->ncols != n || b->nrows != l) return 1;
    if (m == 0 || n == 0 || l == 0) return 0;
    if (k > l) k = (int)l;
    int64_t nstripes = (l + k - 1) / k;
    if (t > nstripes) t = (int)nstripes;
    if (b_s < 1) b_s = m;
    int64_t width = wpr(n), awidth = wpr(l);
    uint64_t atm = tmask(l);
    int kr = (int)(l % k);  /* ragged last stripe width */
    int *slot = (int *)malloc(sizeof(int) << k), *src = (int *)malloc(sizeof(int) << k);
    int *slot_r = NULL, *src_r = NULL;
    gray_steps(k, slot, src);
    if (kr) {
        slot_r = (int *)malloc(sizeof(int) << kr);
        src_r = (int *)malloc(sizeof(int) << kr);
        gray_steps(kr, slot_r, src_r);
    }
    int64_t nblocks = (m + b_s - 1) / b_s;
    int64_t tw = width;
#pragma omp parallel num_threads(g_threads)
    {
        uint64_t *tables = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)t * ((size_t)1 << k) * tw);
        uint64_t *srcbuf = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)k * tw);
        uint64_t *acc = (uint64_t *)malloc(sizeof(uint64_t) * tw);
        int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)t);
#pragma omp for schedule(dynamic, 1)
        for (int64_t blk = 0; blk < nblocks; ++blk) {
            int64_t r0 = blk * b_s, r1 = r0 + b_s < m ? r0 + b_s : m;
            for (int64_t g0 = 0; g0 < nstripes; g0 += t) {
                int gcount = (int)((nstripes - g0) < t ? (nstripes - g0) : t);
                for (int gi = 0; gi < gcount; ++gi) {
                    int64_t sc = (g0 + gi) * k;
                    int kw = (sc + k <= l) ? k : (int)(l - sc);
                    uint64_t *tb = tables + (size_t)gi * ((size_t)1 << k) * tw;
                    if (kw == k) make_table(tb, tw, b, sc, kw, slot, src, srcbuf);
                    else make_table(tb, tw, b, sc, kw, slot_r, src_r, srcbuf);
                }
                for (int64_t r = r0; r < r1; ++r) {
                    const uint64_t *arow = row(a, r);
                    for (int gi = 0; gi < gcount; ++gi) {
                        int64_t sc = (g0 + gi) * k;
                        int kw = (sc + k <= l) ? k : (int)(l - sc);
                        ids[gi] = (int64_t)read_bits(arow, sc, kw, awidth, atm);
                    }
                    const uint64_t *t0 = tables + (size_t)ids[0] * tw;
                    for (int64_t x = 0; x < width; ++x) acc[x] = t0[x];
                    for (int gi = 1; gi < gcount; ++gi) {
                        const uint64_t *tg = tables + (size_t)gi * ((size_t)1 << k) * tw + (size_t)ids[gi] * tw;
                        for (int64_t x = 0; x < width; ++x) acc[x] ^= tg[x];
                    }
                    uint64_t *crow = row(c, r);
                    for (int64_t x = 0; x < width; ++x) crow[x] ^= acc[x];
                }
            }
        }
        free(tables); free(srcbuf); free(acc); free(ids);
    }
    free(slot); free(src); free(slot_r); free(src_r);
    return 0;
}

/* cubic.py:76-102 restated: C[i,j] = parity(A_i & B^T_j) (narrow B). */
static void mul_cubic_into(const omat *c, const omat *a, const omat *b) {
    int64_t m = a->nrows, l = a->ncols, n = b->ncols;
    int64_t lw = wpr(l);
    uint64_t atm = tmask(l);
    uint64_t *bt = (uint64_t *)calloc((size_t)(n * lw) + 1, sizeof(uint64_t));
    for (int64_t kx = 0; kx < l; ++kx) {
        const uint64_t *br = row(b, kx);
        for (int64_t j = 0; j < n; ++j)
            if ((br[j / WB] >> (63 - j % WB)) & 1) bt[j * lw + kx / WB] |= 1ULL << (63 - kx % WB);
    }
    int64_t cw = wpr(n);
    for (int64_t i = 0; i < m; ++i) {
        const uint64_t *ar = row(a, i);
        uint64_t *cr = row(c, i);
        for (int64_t x = 0; x < cw; ++x) cr[x] = 0;
        for (int64_t j = 0; j < n; ++j) {
            uint64_t s = 0;
            for (int64_t x = 0; x < lw; ++x) {
                uint64_t av = ar[x];
                if (x == lw - 1) av &= atm;
                s ^= av & bt[j * lw + x];
            }
            if (__builtin_popcountll(s) & 1) cr[j / WB] |= 1ULL << (63 - j % WB);
        }
    }
    free(bt);
}

/* ------------------------------------------------------------ strassen */
typedef struct { int64_t cutoff, b_s; int k, t; } oparams;

static int eff_k(const oparams *p, int64_t ncols) {
    /* tuning.py:29-44 choose_k(max(b_s,2), l1=32768, t, ncols) when k==0 */
    if (p->k) return p->k;
    int64_t bs = p->b_s < 2 ? 2 : p->b_s;
    int lg = 0;
    double v = 0.75 * __builtin_log2((double)bs);
    int k0 = (int)v - 2;
    (void)lg;
    if (k0 < 1) k0 = 1;
    if (k0 > 16) k0 = 16;
    if (k0 > 1) {
        int64_t row_bytes = wpr(ncols) * 8;
        int fits0 = (int64_t)p->t * (1LL << k0) * row_bytes <= 32768;
        int fits1 = (int64_t)p->t * (1LL << (k0 - 1)) * row_bytes <= 32768;
        if (!fits0 && fits1) return k0 - 1;
    }
    return k0;
}

/* strassen.py:102-123 */
static void base_mul_into(const omat *dst, const omat *a, const omat *b,
                          const oparams *p, int accumulate) {
    int64_t m = a->nrows, l = a->ncols, n = b->ncols;
    if (m == 0 || n == 0) return;
    omat own = owned(m, n);
    if (l == 0 || n < WB) {
        if (l) mul_cubic_into(&own, a, b);
    } else {
        oracle_m4rm_mul_into(&own, a, b, eff_k(p, n), p->b_s, p->t);
    }
    if (accumulate) add_into(dst, dst, &own);
    else copy_into(dst, &own);
    free(own.w);
}

/* strassen.py:141-204: one level, 7 products and 15 adds, 22-step order. */
static void mul_rec(const omat *c, const omat *a, const omat *b, int depth,
                    int max_depth, const oparams *p, omat *arena);

static void schedule_winograd(const omat *a, const omat *b, const omat *c,
                              omat *xbuf, omat *ybuf, int depth, int max_depth,
                              const oparams *p, omat *arena) {
    int64_t m2 = a->nrows / 2, l2 = a->ncols / 2, n2 = b->ncols / 2;
    omat a11 = sub(a, 0, 0, m2, l2), a12 = sub(a, 0, l2, m2, l2);
    omat a21 = sub(a, m2, 0, m2, l2), a22 = sub(a, m2, l2, m2, l2);
    omat b11 = sub(b, 0, 0, l2, n2), b12 = sub(b, 0, n2, l2, n2);
    omat b21 = sub(b, l2, 0, l2, n2), b22 = sub(b, l2, n2, l2, n2);
    omat c11 = sub(c, 0, 0, m2, n2), c12 = sub(c, 0, n2, m2, n2);
    omat c21 = sub(c, m2, 0, m2, n2), c22 = sub(c, m2, n2, m2, n2);
    omat xs = sub(xbuf, 0, 0, m2, l2), xp = sub(xbuf, 0, 0, m2, n2);
    omat y = sub(ybuf, 0, 0, l2, n2);
#define MUL(D, U, V) mul_rec(&(D), &(U), &(V), depth + 1, max_depth, p, arena)
    add_into(&xs, &a11, &a21);
    add_into(&y, &b22, &b12);
    MUL(c21, xs, y);
    add_into(&xs, &a21, &a22);
    add_into(&y, &b12, &b11);
    MUL(c22, xs, y);
    add_into(&xs, &xs, &a11);
    add_into(&y, &b22, &y);
    MUL(c12, xs, y);
    add_into(&xs, &a12, &xs);
    MUL(c11, xs, b22);
    MUL(xp, a11, b11);
    add_into(&c12, &xp, &c12);
    add_into(&c21, &c12, &c21);
    add_into(&c12, &c12, &c22);
    add_into(&c22, &c21, &c22);
    add_into(&c12, &c12, &c11);
    add_into(&y, &y, &b21);
    MUL(c11, a22, y);
    add_into(&c21, &c21, &c11);
    MUL(c11, a12, b21);
    add_into(&c11, &xp, &c11);
#undef MUL
}

static void mul_rec(const omat *c, const omat *a, const omat *b, int depth,
                    int max_depth, const oparams *p, omat *arena) {
    if (depth == max_depth) {
        base_mul_into(c, a, b, p, 0);
        return;
    }
    schedule_winograd(a, b, c, &arena[2 * depth], &arena[2 * depth + 1], depth,
                      max_depth, p, arena);
}

/* strassen.py:66-84 */
void oracle_peel_split(int64_t m, int64_t l, int64_t n, int64_t cutoff, int64_t *out4) {
    out4[0] = out4[1] = out4[2] = out4[3] = 0;
#define OK(d) (((m / (WB << (d))) * WB >= cutoff) && ((l / (WB << (d))) * WB >= cutoff) && \
               ((n / (WB << (d))) * WB >= cutoff))
    if (m < 1 || l < 1 || n < 1 || !OK(1)) return;
    int depth = 1;
    while (depth < 40 && OK(depth + 1)) ++depth;
#undef OK
    int64_t unit = (int64_t)WB << depth;
    out4[0] = (m / unit) * unit;
    out4[1] = (l / unit) * unit;
    out4[2] = (n / unit) * unit;
    out4[3] = depth;
}

/* strassen.py:257-282 (+219-249 peel_fixup). c is overwritten (accumulate=0)
 * or XOR-accumulated (accumulate=1, i.e. add_into(C, C, mul_strassen(A,B))). */
int oracle_mul_strassen(const omat *c_in, const omat *a, const omat *b, int64_t cutoff,
                        int64_t b_s, int k, int t, int accumulate) {
    int64_t m = a->nrows, l = a->ncols, n = b->ncols;
    if (b->nrows != l || c_in->nrows != m || c_in->ncols != n) return 1;
    oparams p = {cutoff, b_s > 0 ? b_s : (cutoff / 2 > 1 ? cutoff / 2 : 1), k, t};
    omat cres = owned(m, n);
    const omat *c = &cres;
    if (m && n && l) {
        int64_t ps[4];
        oracle_peel_split(m, l, n, cutoff, ps);
        if (n < WB) {
            mul_cubic_into(c, a, b);
        } else if ((m < l ? (m < n ? m : n) : (l < n ? l : n)) <= cutoff || ps[3] == 0) {
            oracle_m4rm_mul_into(c, a, b, eff_k(&p, n), p.b_s, p.t);
        } else {
            int depth = (int)ps[3];
            omat *arena = (omat *)malloc(sizeof(omat) * 2 * depth);
            for (int s = 1; s <= depth; ++s) {  /* strassen.py:126-138 */
                int64_t xm = ps[0] >> s, xl = ps[1] >> s, xn = ps[2] >> s;
                arena[2 * (s - 1)] = owned(xm, xl > xn ? xl : xn);
                arena[2 * (s - 1) + 1] = owned(xl, xn);
            }
            omat c0 = sub(c, 0, 0, ps[0], ps[2]), a0 = sub(a, 0, 0, ps[0], ps[1]),
                 b0 = sub(b, 0, 0, ps[1], ps[2]);
            mul_rec(&c0, &a0, &b0, 0, depth, &p, arena);
            for (int s = 0; s < 2 * depth; ++s) free(arena[s].w);
            free(arena);
            int64_t m2 = ps[0], l2 = ps[1], n2 = ps[2];
            if (l2 < l && m2 && n2) {
                omat cc = sub(c, 0, 0, m2, n2), aa = sub(a, 0, l2, m2, l - l2),
                     bb = sub(b, l2, 0, l - l2, n2);
                base_mul_into(&cc, &aa, &bb, &p, 1);
            }
            if (m2 < m) {
                omat cc = sub(c, m2, 0, m - m2, n), aa = sub(a, m2, 0, m - m2, l),
                     bb = sub(b, 0, 0, l, n);
                base_mul_into(&cc, &aa, &bb, &p, 0);
            }
            if (n2 < n) {
                omat cc = sub(c, 0, n2, m2, n - n2), aa = sub(a, 0, 0, m2, l),
                     bb = sub(b, 0, n2, l, n - n2);
                base_mul_into(&cc, &aa, &bb, &p, 0);
            }
        }
    }
    if (accumulate) add_into(c_in, c_in, c);
    else copy_into(c_in, c);
    free(cres.w);
    return 0;
}
