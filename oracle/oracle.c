/*
 * oracle/oracle.c -- the CPU ORACLE of the hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library. The product path (paper_2604_13191_b200/) never imports,
 * links or executes anything under oracle/, and this file shares no code, header,
 * table or constant generator with it.
 *
 * What it computes (paper: "Fast Voxelization and Level of Detail for Microgeometry
 * Rendering", arXiv 2604.13191; P:n = PAPER.md line n, S:n = SPEC.md line n):
 *   - sparse voxelization of fiber segments and triangles into a Morton-keyed grid
 *     (P:164-170 normalisation, P:190-198 block test, P:242-248 gathering),
 *   - per-voxel density mass and SGGX second moment M (moment form),
 *   - the 2x2x2 LoD pyramid with SGGX-H clustering per parent.
 * Formula by formula it follows docs/PREDICATES.md (section numbers "§n" below), which
 * pins every floating-point operation (IEEE binary32, no FMA: compile with
 * -ffp-contract=off and without -ffast-math) so that integer decisions (keys, merge
 * argmins) are taken in the kernel's precision on both sides, and every sum of
 * contributions is an exact integer sum (__int128 here).
 *
 * It is deliberately plain and slow: per primitive it enumerates every candidate voxel,
 * evaluates the predicate, appends (key, quantised contribution) records, then sorts
 * the records by key (qsort) and sums each run. SGGX-H recomputes every sigma and the
 * full distance matrix after every merge.
 *
 * Parity pins (tests/test_oracle_*.py): closed forms (axis-aligned rectangle key
 * counts, straight-fiber key sets and lengths), fp64 shadows, exact-rational SAT,
 * brute force over all N^3 voxels, conservation laws, SPEC worked examples
 * (tests/golden/). "Parity unpinned": the choice of the fiber
 * weight l_r and of the sigma-distance have no printed value in the paper to match.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

#define ORC_OK 0
#define ORC_ERR_ARG -1
#define ORC_ERR_OOM -2
#define ORC_ERR_OVERFLOW -3
#define ORC_ERR_LEVEL -4

#define MAX_LEVELS 14
#define MAX_K 8

/* ------------------------------------------------------------------ small helpers */

static float fminf_(float a, float b) { return a < b ? a : b; }
static float fmaxf_(float a, float b) { return a > b ? a : b; }

/* §8: q(x) = llrint(fl(x * 2^32)) */
static int64_t q32(float x) {
    float y = x * 4294967296.0f;
    return llrintf(y);
}

/* §8: fp32 output = fl((float)acc * 2^-32); acc must fit int64 (checked by caller). */
static float deq32(i128 acc) {
    float f = (float)(int64_t)acc;
    return f * 2.3283064365386963e-10f; /* 2^-32, exact */
}

static int fits64(i128 v) { return v >= (i128)INT64_MIN && v <= (i128)INT64_MAX; }

/* §2 Morton key, x in bit 0 */
uint64_t orc_morton(uint32_t i, uint32_t j, uint32_t k) {
    uint64_t key = 0;
    for (int b = 0; b < 21; b++) {
        key |= (uint64_t)((i >> b) & 1u) << (3 * b);
        key |= (uint64_t)((j >> b) & 1u) << (3 * b + 1);
        key |= (uint64_t)((k >> b) & 1u) << (3 * b + 2);
    }
    return key;
}

void orc_unmorton(uint64_t key, uint32_t* i, uint32_t* j, uint32_t* k) {
    uint32_t x = 0, y = 0, z = 0;
    for (int b = 0; b < 21; b++) {
        x |= (uint32_t)((key >> (3 * b)) & 1u) << b;
        y |= (uint32_t)((key >> (3 * b + 1)) & 1u) << b;
        z |= (uint32_t)((key >> (3 * b + 2)) & 1u) << b;
    }
    *i = x; *j = y; *k = z;
}

/* ------------------------------------------------------------------ §1 grid transform */

typedef struct {
    uint32_t N;
    float bmin[3];
    float E;
    float Nf;
} grid_t;

static int grid_init(grid_t* g, uint32_t N, const float bbox[6]) {
    if (N < 2 || N > 8192 || (N & (N - 1))) return ORC_ERR_ARG;
    float e[3];
    for (int a = 0; a < 3; a++) {
        if (!isfinite(bbox[a]) || !isfinite(bbox[3 + a])) return ORC_ERR_ARG;
        e[a] = bbox[3 + a] - bbox[a];
        if (!(e[a] > 0.0f)) return ORC_ERR_ARG;
        g->bmin[a] = bbox[a];
    }
    g->E = fmaxf_(fmaxf_(e[0], e[1]), e[2]);
    g->N = N;
    g->Nf = (float)N;
    return ORC_OK;
}

static float grid_coord(const grid_t* g, int a, float p) {
    float t = p - g->bmin[a];
    t = t / g->E;
    return t * g->Nf;
}

static float grid_len(const grid_t* g, float r) {
    float t = r / g->E;
    return t * g->Nf;
}

void orc_grid(const float bbox[6], uint32_t N, const float p[3], float out[3]) {
    grid_t g;
    if (grid_init(&g, N, bbox) != ORC_OK) { out[0] = out[1] = out[2] = NAN; return; }
    for (int a = 0; a < 3; a++) out[a] = grid_coord(&g, a, p[a]);
}

/* ------------------------------------------------------------------ §4 fiber predicate */

typedef struct {
    float a[3];      /* grid-space start */
    float d[3];      /* fl(b - a) */
    float w[3];      /* fl(d*d) */
    float iota[3];   /* fl(1/d) for moving axes */
    int moving[3];
    float r2;        /* fl(rg*rg) */
    float len;       /* |d| */
} fiber_t;

static void fiber_setup(fiber_t* f, const float a[3], const float b[3], float rg) {
    for (int ax = 0; ax < 3; ax++) {
        f->a[ax] = a[ax];
        f->d[ax] = b[ax] - a[ax];
        f->w[ax] = f->d[ax] * f->d[ax];
        f->moving[ax] = f->w[ax] > 0.0f;
        f->iota[ax] = f->moving[ax] ? 1.0f / f->d[ax] : 0.0f;
    }
    f->r2 = rg * rg;
    float s = f->w[0] + f->w[1];
    s = s + f->w[2];
    f->len = sqrtf(s);
}

/* Returns 1 iff voxel (i,j,k) is a key of the capsule; then *ell = l_r (§4). */
static int fiber_eval(const fiber_t* f, int64_t i, int64_t j, int64_t k, float* ell) {
    const float lo[3] = {(float)i, (float)j, (float)k};
    const float hi[3] = {(float)(i + 1), (float)(j + 1), (float)(k + 1)};
    float u[3] = {0, 0, 0}, v[3] = {0, 0, 0};
    float Wu[3] = {0, 0, 0}, Wuu[3] = {0, 0, 0}, Wv[3] = {0, 0, 0}, Wvv[3] = {0, 0, 0};
    float C0 = 0.0f;
    float bp[8];
    int nbp = 0;
    bp[nbp++] = 0.0f;
    for (int ax = 0; ax < 3; ax++) {
        if (f->moving[ax]) {
            float t1 = (lo[ax] - f->a[ax]) * f->iota[ax];
            float t2 = (hi[ax] - f->a[ax]) * f->iota[ax];
            u[ax] = fminf_(t1, t2);
            v[ax] = fmaxf_(t1, t2);
            Wu[ax] = f->w[ax] * u[ax];
            Wuu[ax] = Wu[ax] * u[ax];
            Wv[ax] = f->w[ax] * v[ax];
            Wvv[ax] = Wv[ax] * v[ax];
            if (u[ax] > 0.0f && u[ax] < 1.0f) bp[nbp++] = u[ax];
            if (v[ax] > 0.0f && v[ax] < 1.0f) bp[nbp++] = v[ax];
        } else {
            float c = 0.0f;
            if (f->a[ax] < lo[ax]) c = lo[ax] - f->a[ax];
            else if (f->a[ax] > hi[ax]) c = f->a[ax] - hi[ax];
            C0 = C0 + c * c;
        }
    }
    /* sort the interior breakpoints (indices 1..nbp-1) ascending; then append 1 */
    for (int x = 2; x < nbp; x++) {
        float key = bp[x];
        int y = x - 1;
        while (y >= 1 && bp[y] > key) { bp[y + 1] = bp[y]; y--; }
        bp[y + 1] = key;
    }
    bp[nbp++] = 1.0f;

    int found = 0;
    float ta = 0.0f, tb = 0.0f;
    for (int m = 0; m + 1 < nbp; m++) {
        float L = bp[m], H = bp[m + 1];
        float A = 0.0f, B = 0.0f, C = C0;
        for (int ax = 0; ax < 3; ax++) {
            if (!f->moving[ax]) continue;
            if (u[ax] >= H) { A = A + f->w[ax]; B = B + Wu[ax]; C = C + Wuu[ax]; }
            else if (v[ax] <= L) { A = A + f->w[ax]; B = B + Wv[ax]; C = C + Wvv[ax]; }
        }
        float lo_m, hi_m;
        if (A == 0.0f) {
            if (!(C <= f->r2)) continue;
            lo_m = L; hi_m = H;
        } else {
            float Cr = C - f->r2;
            float D = B * B - A * Cr;   /* two fl products then one fl difference */
            if (D < 0.0f) continue;
            float s = sqrtf(D);
            float t1 = (B - s) / A;
            float t2 = (B + s) / A;
            lo_m = fmaxf_(t1, L);
            hi_m = fminf_(t2, H);
            if (!(lo_m <= hi_m)) continue;
        }
        if (!found) { ta = lo_m; tb = hi_m; found = 1; }
        else { ta = fminf_(ta, lo_m); tb = fmaxf_(tb, hi_m); }
    }
    if (!found) return 0;
    *ell = f->len * (tb - ta);
    return 1;
}

/* Unit entry for tests: grid-space endpoints a, b and grid radius rg. */
int orc_fiber_eval(const float a[3], const float b[3], float rg, int64_t i, int64_t j, int64_t k,
                   float* ell) {
    fiber_t f;
    fiber_setup(&f, a, b, rg);
    float e = 0.0f;
    int key = fiber_eval(&f, i, j, k, &e);
    *ell = e;
    return key;
}

/* ------------------------------------------------------------------ §6 triangle SAT */

static void cross3(const float f[3], const float g[3], float out[3]) {
    out[0] = f[1] * g[2] - f[2] * g[1];
    out[1] = f[2] * g[0] - f[0] * g[2];
    out[2] = f[0] * g[1] - f[1] * g[0];
}

static int sep3(float p0, float p1, float p2, float rad) {
    float mn = fminf_(fminf_(p0, p1), p2);
    float mx = fmaxf_(fmaxf_(p0, p1), p2);
    return mn > rad || mx < -rad;
}

static int tri_sat(const float g[9], int64_t i, int64_t j, int64_t k) {
    const float h = 0.5f;
    const float c[3] = {(float)i + 0.5f, (float)j + 0.5f, (float)k + 0.5f};
    float v[3][3], e[3][3];
    for (int m = 0; m < 3; m++)
        for (int ax = 0; ax < 3; ax++) v[m][ax] = g[3 * m + ax] - c[ax];
    for (int ax = 0; ax < 3; ax++) {
        e[0][ax] = v[1][ax] - v[0][ax];
        e[1][ax] = v[2][ax] - v[1][ax];
        e[2][ax] = v[0][ax] - v[2][ax];
    }
    for (int q = 0; q < 3; q++) {
        const float ex = e[q][0], ey = e[q][1], ez = e[q][2];
        const float fx = fabsf(ex), fy = fabsf(ey), fz = fabsf(ez);
        float p[3], rad;
        /* X axis */
        for (int m = 0; m < 3; m++) p[m] = ez * v[m][1] - ey * v[m][2];
        rad = fz * h + fy * h;
        if (sep3(p[0], p[1], p[2], rad)) return 0;
        /* Y axis */
        for (int m = 0; m < 3; m++) p[m] = ex * v[m][2] - ez * v[m][0];
        rad = fz * h + fx * h;
        if (sep3(p[0], p[1], p[2], rad)) return 0;
        /* Z axis */
        for (int m = 0; m < 3; m++) p[m] = ey * v[m][0] - ex * v[m][1];
        rad = fy * h + fx * h;
        if (sep3(p[0], p[1], p[2], rad)) return 0;
    }
    for (int ax = 0; ax < 3; ax++) {
        float mn = fminf_(fminf_(v[0][ax], v[1][ax]), v[2][ax]);
        float mx = fmaxf_(fmaxf_(v[0][ax], v[1][ax]), v[2][ax]);
        if (mn > h || mx < -h) return 0;
    }
    float n[3], vmin[3], vmax[3];
    cross3(e[0], e[1], n);
    for (int ax = 0; ax < 3; ax++) {
        if (n[ax] > 0.0f) { vmin[ax] = -h - v[0][ax]; vmax[ax] = h - v[0][ax]; }
        else { vmin[ax] = h - v[0][ax]; vmax[ax] = -h - v[0][ax]; }
    }
    float dmin = n[0] * vmin[0] + n[1] * vmin[1];
    dmin = dmin + n[2] * vmin[2];
    if (dmin > 0.0f) return 0;
    float dmax = n[0] * vmax[0] + n[1] * vmax[1];
    dmax = dmax + n[2] * vmax[2];
    if (dmax < 0.0f) return 0;
    return 1;
}

int orc_tri_sat(const float g[9], int64_t i, int64_t j, int64_t k) { return tri_sat(g, i, j, k); }

/* ------------------------------------------------------------------ §7 clipped area */

#define MAXPOLY 12

static int clip_plane(float in[][3], int n, float out[][3], int ax, float c, int upper) {
    int m_out = 0;
    for (int m = 0; m < n; m++) {
        const float* cur = in[m];
        const float* prev = in[(m + n - 1) % n];
        int cin = upper ? (cur[ax] < c) : (cur[ax] >= c);
        int pin = upper ? (prev[ax] < c) : (prev[ax] >= c);
        if (cin != pin) {
            /* I(prev, cur) */
            float s = (c - prev[ax]) / (cur[ax] - prev[ax]);
            for (int b = 0; b < 3; b++) {
                if (b == ax) out[m_out][b] = c;
                else out[m_out][b] = prev[b] + s * (cur[b] - prev[b]);
            }
            m_out++;
        }
        if (cin) {
            for (int b = 0; b < 3; b++) out[m_out][b] = cur[b];
            m_out++;
        }
    }
    return m_out;
}

static float tri_area_in(const float g[9], int64_t i, int64_t j, int64_t k) {
    float P[MAXPOLY][3], Q[MAXPOLY][3];
    for (int m = 0; m < 3; m++)
        for (int ax = 0; ax < 3; ax++) P[m][ax] = g[3 * m + ax];
    int n = 3;
    const float lo[3] = {(float)i, (float)j, (float)k};
    const float hi[3] = {(float)(i + 1), (float)(j + 1), (float)(k + 1)};
    for (int ax = 0; ax < 3; ax++) {
        n = clip_plane(P, n, Q, ax, lo[ax], 0);
        if (n < 3) return 0.0f;
        n = clip_plane(Q, n, P, ax, hi[ax], 1);
        if (n < 3) return 0.0f;
    }
    float acc[3] = {0.0f, 0.0f, 0.0f};
    for (int m = 1; m + 1 < n; m++) {
        float e1[3], e2[3], cr[3];
        for (int ax = 0; ax < 3; ax++) {
            e1[ax] = P[m][ax] - P[0][ax];
            e2[ax] = P[m + 1][ax] - P[0][ax];
        }
        cross3(e1, e2, cr);
        for (int ax = 0; ax < 3; ax++) acc[ax] = acc[ax] + cr[ax];
    }
    float s = acc[0] * acc[0] + acc[1] * acc[1];
    s = s + acc[2] * acc[2];
    return 0.5f * sqrtf(s);
}

float orc_tri_area(const float g[9], int64_t i, int64_t j, int64_t k) { return tri_area_in(g, i, j, k); }

/* ------------------------------------------------------------------ records, levels */

typedef struct {
    uint64_t key;
    int64_t q[7];
} rec_t;

typedef struct {
    uint64_t n;
    uint64_t* key;
    i128* acc;      /* [n][7] */
    uint8_t* ncl;   /* [n] */
    i128* cl;       /* [n][K][7] */
} level_t;

/* §10 tables (histogram distance mode), defined with the §10 code below */
#define HIST_BINS 125
#define HIST_NMIN 32
#define HIST_NMAX 8160
typedef struct hist_tables {
    int N;
    float (*u)[3];
    uint8_t perm[32][HIST_BINS];
    int64_t gap[32][HIST_BINS - 1];
} hist_tables_t;

typedef struct {
    grid_t g;
    int logN;
    int K;
    /* emission window: a Morton cell (level wl, index wc) as a voxel box */
    int64_t wlo[3], whi[3];   /* inclusive voxel range */
    rec_t* recs;
    size_t nrec, cap;
    int built;                /* levels built (-1: nothing) */
    level_t lv[MAX_LEVELS];
    int mode;                 /* 0: sigma distance (§9), 1: histogram distance (§10) */
    int hist_n;               /* N samples per histogram (§10) */
    struct hist_tables* ht;   /* §10 tables (mode 1) */
    uint64_t* dm0;            /* §13 level-0 sub-voxel masks [lv[0].n][8] (NULL: none) */
    uint64_t dm0_n;
} orc_ctx;

static int hist_tables_init(hist_tables_t* T, int N);

static int push_rec(orc_ctx* c, uint64_t key, const int64_t q[7]) {
    if (c->nrec == c->cap) {
        size_t nc = c->cap ? 2 * c->cap : 1024;
        rec_t* r = (rec_t*)realloc(c->recs, nc * sizeof(rec_t));
        if (!r) return ORC_ERR_OOM;
        c->recs = r;
        c->cap = nc;
    }
    c->recs[c->nrec].key = key;
    memcpy(c->recs[c->nrec].q, q, sizeof(int64_t) * 7);
    c->nrec++;
    return ORC_OK;
}

static void free_levels(orc_ctx* c) {
    for (int l = 0; l < MAX_LEVELS; l++) {
        free(c->lv[l].key); free(c->lv[l].acc); free(c->lv[l].ncl); free(c->lv[l].cl);
        memset(&c->lv[l], 0, sizeof(level_t));
    }
    c->built = -1;
}

orc_ctx* orc_create(uint32_t N, const float bbox[6], int K) {
    orc_ctx* c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
    if (!c) return NULL;
    if (grid_init(&c->g, N, bbox) != ORC_OK || K < 1 || K > MAX_K) { free(c); return NULL; }
    c->logN = 0;
    while ((1u << c->logN) < N) c->logN++;
    c->K = K;
    for (int a = 0; a < 3; a++) { c->wlo[a] = 0; c->whi[a] = (int64_t)N - 1; }
    c->built = -1;
    c->mode = 0;
    c->hist_n = 5000;
    return c;
}

/* §10: select the SGGX-H distance (0 sigma, 1 histogram with N samples per SGGX) */
int orc_set_distance(orc_ctx* c, int mode, int N) {
    if (mode < 0 || mode > 1 || N < HIST_NMIN || N > HIST_NMAX) return ORC_ERR_ARG;
    if (mode == 1 && (!c->ht || c->ht->N != N)) {
        if (c->ht) { free(c->ht->u); free(c->ht); c->ht = NULL; }
        c->ht = (hist_tables_t*)calloc(1, sizeof(hist_tables_t));
        if (!c->ht) return ORC_ERR_OOM;
        int rc = hist_tables_init(c->ht, N);
        if (rc != ORC_OK) { free(c->ht); c->ht = NULL; return rc; }
    }
    c->mode = mode;
    c->hist_n = N;
    return ORC_OK;
}

void orc_destroy(orc_ctx* c) {
    if (!c) return;
    free_levels(c);
    free(c->recs);
    if (c->ht) { free(c->ht->u); free(c->ht); }
    free(c->dm0);
    free(c);
}

/* Restrict emission to the voxels of Morton cell `cell` at level `wl` (windowed parity).
 * Segment normalisation S_p still runs over all keys (§5), so in-window values are the
 * same as in a full run. */
int orc_set_window(orc_ctx* c, int wl, uint64_t cell) {
    if (wl < 0 || wl > c->logN) return ORC_ERR_ARG;
    uint32_t i, j, k;
    orc_unmorton(cell, &i, &j, &k);
    int64_t sz = (int64_t)1 << wl;
    int64_t o[3] = {(int64_t)i * sz, (int64_t)j * sz, (int64_t)k * sz};
    for (int a = 0; a < 3; a++) {
        if (o[a] + sz > (int64_t)c->g.N) return ORC_ERR_ARG;
        c->wlo[a] = o[a];
        c->whi[a] = o[a] + sz - 1;
    }
    return ORC_OK;
}

static int in_window(const orc_ctx* c, int64_t i, int64_t j, int64_t k) {
    return i >= c->wlo[0] && i <= c->whi[0] && j >= c->wlo[1] && j <= c->whi[1] &&
           k >= c->wlo[2] && k <= c->whi[2];
}

/* §3: integer candidate range [ceil(lo)-1, floor(hi)] of one axis */
static void cand_range(float lo, float hi, int64_t* c0, int64_t* c1) {
    *c0 = (int64_t)ceilf(lo) - 1;
    *c1 = (int64_t)floorf(hi);
}

/* §4, §5 */
int orc_add_fibers(orc_ctx* c, const float* seg, const float* radii, uint64_t S) {
    const float PI_F = 3.14159274101257324f; /* 0x40490FDB */
    c->built = -1;
    for (uint64_t p = 0; p < S; p++) {
        const float* s = seg + 6 * p;
        float r = radii[p];
        for (int q = 0; q < 6; q++) if (!isfinite(s[q])) return ORC_ERR_ARG;
        if (!isfinite(r) || r < 0.0f) return ORC_ERR_ARG;
        float a[3], b[3];
        for (int ax = 0; ax < 3; ax++) {
            a[ax] = grid_coord(&c->g, ax, s[ax]);
            b[ax] = grid_coord(&c->g, ax, s[3 + ax]);
        }
        float rg = grid_len(&c->g, r);
        int64_t u0[3], u1[3];   /* unclamped candidate range */
        int culled = 0;
        for (int ax = 0; ax < 3; ax++) {
            float lo = fminf_(a[ax], b[ax]) - rg;
            float hi = fmaxf_(a[ax], b[ax]) + rg;
            if (!(hi >= -1.0f) || !(lo <= (float)c->g.N + 1.0f)) { culled = 1; break; }
            if (hi - lo > 16777216.0f) return ORC_ERR_ARG; /* > 2^24 candidates (§3) */
            cand_range(lo, hi, &u0[ax], &u1[ax]);
            int64_t e0 = u0[ax] < c->wlo[ax] ? c->wlo[ax] : u0[ax];
            int64_t e1 = u1[ax] > c->whi[ax] ? c->whi[ax] : u1[ax];
            if (e0 > e1) culled = 1;
        }
        if (culled) continue;
        uint64_t ncand = (uint64_t)(u1[0] - u0[0] + 1) * (uint64_t)(u1[1] - u0[1] + 1) *
                         (uint64_t)(u1[2] - u0[2] + 1);
        if (ncand > (1ull << 24)) return ORC_ERR_ARG;
        fiber_t f;
        fiber_setup(&f, a, b, rg);
        /* first pass: every key in the unclamped range -> S_acc */
        float* ells = (float*)malloc(sizeof(float) * ncand);
        uint8_t* iskey = (uint8_t*)malloc(ncand);
        if (!ells || !iskey) { free(ells); free(iskey); return ORC_ERR_OOM; }
        i128 Sacc = 0;
        uint64_t idx = 0;
        for (int64_t k = u0[2]; k <= u1[2]; k++)
            for (int64_t j = u0[1]; j <= u1[1]; j++)
                for (int64_t i = u0[0]; i <= u1[0]; i++, idx++) {
                    float ell = 0.0f;
                    iskey[idx] = (uint8_t)fiber_eval(&f, i, j, k, &ell);
                    ells[idx] = ell;
                    if (iskey[idx]) Sacc += q32(ell);
                }
        if (!fits64(Sacc)) { free(ells); free(iskey); return ORC_ERR_OVERFLOW; }
        float Sp = deq32(Sacc);
        float mp = PI_F * rg;
        mp = mp * rg;
        mp = mp * f.len;
        float fp = Sacc > 0 ? mp / Sp : 0.0f;
        float t[3];
        for (int ax = 0; ax < 3; ax++) t[ax] = f.len > 0.0f ? f.d[ax] / f.len : 0.0f;
        /* second pass: contributions of in-grid, in-window keys */
        idx = 0;
        for (int64_t k = u0[2]; k <= u1[2]; k++)
            for (int64_t j = u0[1]; j <= u1[1]; j++)
                for (int64_t i = u0[0]; i <= u1[0]; i++, idx++) {
                    if (!iskey[idx] || !in_window(c, i, j, k)) continue;
                    float mass = fp * ells[idx];
                    int64_t q[7];
                    q[0] = q32(mass);
                    q[1] = q32((mass * t[0]) * t[0]);
                    q[2] = q32((mass * t[1]) * t[1]);
                    q[3] = q32((mass * t[2]) * t[2]);
                    q[4] = q32((mass * t[0]) * t[1]);
                    q[5] = q32((mass * t[0]) * t[2]);
                    q[6] = q32((mass * t[1]) * t[2]);
                    int rc = push_rec(c, orc_morton((uint32_t)i, (uint32_t)j, (uint32_t)k), q);
                    if (rc) { free(ells); free(iskey); return rc; }
                }
        free(ells);
        free(iskey);
    }
    return ORC_OK;
}

/* §6, §7 */
int orc_add_triangles(orc_ctx* c, const float* tri, const float* dirs, uint64_t T) {
    c->built = -1;
    for (uint64_t t = 0; t < T; t++) {
        const float* v = tri + 9 * t;
        for (int q = 0; q < 9; q++) if (!isfinite(v[q])) return ORC_ERR_ARG;
        float g[9];
        for (int m = 0; m < 3; m++)
            for (int ax = 0; ax < 3; ax++) g[3 * m + ax] = grid_coord(&c->g, ax, v[3 * m + ax]);
        /* direction (face normal of the grid-space triangle, or the caller's dirs) */
        float w[3];
        if (dirs) {
            for (int ax = 0; ax < 3; ax++) {
                w[ax] = dirs[3 * t + ax];
                if (!isfinite(w[ax])) return ORC_ERR_ARG;
            }
        } else {
            float f1[3], f2[3];
            for (int ax = 0; ax < 3; ax++) { f1[ax] = g[3 + ax] - g[ax]; f2[ax] = g[6 + ax] - g[3 + ax]; }
            cross3(f1, f2, w);
        }
        float nn = w[0] * w[0] + w[1] * w[1];
        nn = nn + w[2] * w[2];
        float nrm = sqrtf(nn);
        if (dirs && !(nrm > 0.0f)) return ORC_ERR_ARG;
        float dh[3];
        for (int ax = 0; ax < 3; ax++) dh[ax] = nrm > 0.0f ? w[ax] / nrm : 0.0f;
        int64_t e0[3], e1[3];
        int culled = 0;
        for (int ax = 0; ax < 3; ax++) {
            float lo = fminf_(fminf_(g[ax], g[3 + ax]), g[6 + ax]);
            float hi = fmaxf_(fmaxf_(g[ax], g[3 + ax]), g[6 + ax]);
            if (!(hi >= -1.0f) || !(lo <= (float)c->g.N + 1.0f)) { culled = 1; break; }
            cand_range(lo, hi, &e0[ax], &e1[ax]);
            if (e0[ax] < c->wlo[ax]) e0[ax] = c->wlo[ax];
            if (e1[ax] > c->whi[ax]) e1[ax] = c->whi[ax];
            if (e0[ax] > e1[ax]) culled = 1;
        }
        if (culled) continue;
        for (int64_t k = e0[2]; k <= e1[2]; k++)
            for (int64_t j = e0[1]; j <= e1[1]; j++)
                for (int64_t i = e0[0]; i <= e1[0]; i++) {
                    if (!tri_sat(g, i, j, k)) continue;
                    float A = tri_area_in(g, i, j, k);
                    float mass = 1.0f * A;
                    int64_t q[7];
                    q[0] = q32(mass);
                    q[1] = q32((mass * dh[0]) * dh[0]);
                    q[2] = q32((mass * dh[1]) * dh[1]);
                    q[3] = q32((mass * dh[2]) * dh[2]);
                    q[4] = q32((mass * dh[0]) * dh[1]);
                    q[5] = q32((mass * dh[0]) * dh[2]);
                    q[6] = q32((mass * dh[1]) * dh[2]);
                    int rc = push_rec(c, orc_morton((uint32_t)i, (uint32_t)j, (uint32_t)k), q);
                    if (rc) return rc;
                }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ §12 sampling front end */
/* The paper's own voxelization: Catmull-Rom spline pieces sampled at
 * t_s = (s + 1/2)/n and triangles sampled with Heitz's low-distortion map,
 * sample counts proportional to area; each sample adds to the voxel containing it. */
static int push_sample(orc_ctx* c, const float p[3], float f, const float d[3]) {
    int64_t v[3];
    for (int ax = 0; ax < 3; ax++) {
        float fl_ = floorf(p[ax]);
        if (!(fl_ >= 0.0f) || !(fl_ < (float)c->g.N)) return ORC_OK; /* outside [0, N): dropped */
        v[ax] = (int64_t)fl_;
    }
    if (!in_window(c, v[0], v[1], v[2])) return ORC_OK;
    int64_t q[7];
    q[0] = q32(f);
    q[1] = q32((f * d[0]) * d[0]);
    q[2] = q32((f * d[1]) * d[1]);
    q[3] = q32((f * d[2]) * d[2]);
    q[4] = q32((f * d[0]) * d[1]);
    q[5] = q32((f * d[0]) * d[2]);
    q[6] = q32((f * d[1]) * d[2]);
    return push_rec(c, orc_morton((uint32_t)v[0], (uint32_t)v[1], (uint32_t)v[2]), q);
}

/* position and unit tangent of a grid-space Catmull-Rom piece at t (§12) */
static void spline_eval(const float G[4][3], float t, float pos[3], float tan_[3]) {
    float dv[3];
    for (int ax = 0; ax < 3; ax++) {
        float c0 = 2.0f * G[1][ax];
        float c1 = G[2][ax] - G[0][ax];
        float c2 = ((2.0f * G[0][ax] - 5.0f * G[1][ax]) + 4.0f * G[2][ax]) - G[3][ax];
        float c3 = ((3.0f * G[1][ax] - G[0][ax]) - 3.0f * G[2][ax]) + G[3][ax];
        pos[ax] = 0.5f * (((c3 * t + c2) * t + c1) * t + c0);
        dv[ax] = 0.5f * ((3.0f * c3 * t + 2.0f * c2) * t + c1);
    }
    float nn = dv[0] * dv[0] + dv[1] * dv[1];
    nn = nn + dv[2] * dv[2];
    float nrm = sqrtf(nn);
    for (int ax = 0; ax < 3; ax++) tan_[ax] = nrm > 0.0f ? dv[ax] / nrm : 0.0f;
}

void orc_spline_eval(const float G[12], float t, float pos[3], float tan_[3]) {
    spline_eval((const float(*)[3])G, t, pos, tan_);
}

int orc_sample_splines(orc_ctx* c, const float* ctrl, const float* radii, uint64_t S, int n) {
    const float PI_F = 3.14159274101257324f;
    if (n < 1) return ORC_ERR_ARG;
    c->built = -1;
    for (uint64_t p = 0; p < S; p++) {
        float G[4][3];
        for (int m = 0; m < 4; m++)
            for (int ax = 0; ax < 3; ax++) {
                float w = ctrl[12 * p + 3 * m + ax];
                if (!isfinite(w)) return ORC_ERR_ARG;
                G[m][ax] = grid_coord(&c->g, ax, w);
            }
        float r = radii[p];
        if (!isfinite(r) || r < 0.0f) return ORC_ERR_ARG;
        float rg = grid_len(&c->g, r);
        float d[3] = {G[2][0] - G[1][0], G[2][1] - G[1][1], G[2][2] - G[1][2]};
        float dd = d[0] * d[0] + d[1] * d[1];
        dd = dd + d[2] * d[2];
        float mp = PI_F * rg;
        mp = mp * rg;
        mp = mp * sqrtf(dd);
        float f = mp / (float)n;
        for (int s = 0; s < n; s++) {
            float t = ((float)s + 0.5f) / (float)n;
            float pos[3], tan_[3];
            spline_eval((const float(*)[3])G, t, pos, tan_);
            int rc = push_sample(c, pos, f, tan_);
            if (rc) return rc;
        }
    }
    return ORC_OK;
}

/* whole-triangle area (§7 area formula, one fan term) and direction (§7) in grid space */
static float tri_whole_area(const float g[9]) {
    float e1[3], e2[3], cr[3];
    for (int ax = 0; ax < 3; ax++) { e1[ax] = g[3 + ax] - g[ax]; e2[ax] = g[6 + ax] - g[ax]; }
    cross3(e1, e2, cr);
    float acc[3] = {0.0f + cr[0], 0.0f + cr[1], 0.0f + cr[2]};
    float nn = acc[0] * acc[0] + acc[1] * acc[1];
    nn = nn + acc[2] * acc[2];
    return 0.5f * sqrtf(nn);
}

int orc_tri_samples(float A, float Amax, int budget) {
    if (!(A > 0.0f)) return 0;
    int k = (int)floorf((A / Amax) * (float)budget + 0.5f);
    return k < 1 ? 1 : k;
}

void orc_tri_uv(int s, int n, float* u0, float* u1) {
    *u0 = ((float)s + 0.5f) / (float)n;
    float x = (float)s * 0.618034f;
    *u1 = x - floorf(x);
}

/* unit entry for tests: the n sample points (grid space) of one grid-space triangle */
void orc_tri_sample_points(const float g[9], int n, float* out) {
    for (int s = 0; s < n; s++) {
        float u0, u1, b0, b1;
        orc_tri_uv(s, n, &u0, &u1);
        if (u1 > u0) { b0 = 0.5f * u0; b1 = u1 - b0; }
        else { b1 = 0.5f * u1; b0 = u0 - b1; }
        float b2 = (1.0f - b0) - b1;
        for (int ax = 0; ax < 3; ax++) out[3 * s + ax] = (b0 * g[ax] + b1 * g[3 + ax]) + b2 * g[6 + ax];
    }
}

int orc_sample_triangles(orc_ctx* c, const float* tri, const float* dirs, uint64_t T, int budget) {
    if (budget < 1) return ORC_ERR_ARG;
    c->built = -1;
    float Amax = 0.0f;
    for (uint64_t t = 0; t < T; t++) {
        float g[9];
        for (int q = 0; q < 9; q++) {
            if (!isfinite(tri[9 * t + q])) return ORC_ERR_ARG;
            g[q] = grid_coord(&c->g, q % 3, tri[9 * t + q]);
        }
        float A = tri_whole_area(g);
        if (A > Amax) Amax = A;
    }
    for (uint64_t t = 0; t < T; t++) {
        float g[9];
        for (int q = 0; q < 9; q++) g[q] = grid_coord(&c->g, q % 3, tri[9 * t + q]);
        float w[3];
        if (dirs) {
            for (int ax = 0; ax < 3; ax++) {
                w[ax] = dirs[3 * t + ax];
                if (!isfinite(w[ax])) return ORC_ERR_ARG;
            }
        } else {
            float f1[3], f2[3];
            for (int ax = 0; ax < 3; ax++) { f1[ax] = g[3 + ax] - g[ax]; f2[ax] = g[6 + ax] - g[3 + ax]; }
            cross3(f1, f2, w);
        }
        float nn = w[0] * w[0] + w[1] * w[1];
        nn = nn + w[2] * w[2];
        float nrm = sqrtf(nn);
        if (dirs && !(nrm > 0.0f)) return ORC_ERR_ARG;
        float dh[3];
        for (int ax = 0; ax < 3; ax++) dh[ax] = nrm > 0.0f ? w[ax] / nrm : 0.0f;
        float A = tri_whole_area(g);
        int nt = orc_tri_samples(A, Amax, budget);
        if (nt == 0) continue;
        float f = A / (float)nt;
        for (int s = 0; s < nt; s++) {
            float u0, u1, b0, b1;
            orc_tri_uv(s, nt, &u0, &u1);
            if (u1 > u0) { b0 = 0.5f * u0; b1 = u1 - b0; }
            else { b1 = 0.5f * u1; b0 = u0 - b1; }
            float b2 = (1.0f - b0) - b1;
            float p[3];
            for (int ax = 0; ax < 3; ax++) p[ax] = (b0 * g[ax] + b1 * g[3 + ax]) + b2 * g[6 + ax];
            int rc = push_sample(c, p, f, dh);
            if (rc) return rc;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ §13 sub-voxel density */
/* The paper's occupancy and axis-projected densities:
 * Res_3 = 8 sub-voxels per voxel edge; sub-voxel (a,b,c) of voxel (i,j,k) is hit iff the key
 * predicate of §4 / §6 holds for the fine voxel (8i+a, 8j+b, 8k+c) with grid-space geometry
 * scaled by 8 (exactly the key predicate of an 8N grid). Masks are OR-ed over primitives. */
static int64_t key_index(const level_t* L, uint64_t key) {
    int64_t lo = 0, hi = (int64_t)L->n - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (L->key[mid] == key) return mid;
        if (L->key[mid] < key) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

static int density_prepare(orc_ctx* c) {
    if (c->built < 0) return ORC_ERR_LEVEL;
    if (!c->dm0 || c->dm0_n != c->lv[0].n) {
        free(c->dm0);
        c->dm0_n = c->lv[0].n;
        c->dm0 = (uint64_t*)calloc((c->dm0_n ? c->dm0_n : 1) * 8, sizeof(uint64_t));
        if (!c->dm0) return ORC_ERR_OOM;
    }
    return ORC_OK;
}

static void density_set(orc_ctx* c, int64_t x, int64_t y, int64_t z) {
    int64_t v = key_index(&c->lv[0], orc_morton((uint32_t)(x >> 3), (uint32_t)(y >> 3), (uint32_t)(z >> 3)));
    if (v < 0) return; /* a fine hit outside the key set (possible only by rounding): dropped */
    c->dm0[8 * v + (z & 7)] |= 1ull << ((x & 7) + 8 * (y & 7));
}

/* fine candidate range of one axis, clamped to the grid and the window */
static int fine_range(const orc_ctx* c, int ax, float lo, float hi, int64_t* f0, int64_t* f1) {
    int64_t N8 = 8 * (int64_t)c->g.N;
    if (!(hi >= -1.0f) || !(lo <= (float)N8 + 1.0f)) return 0;
    cand_range(lo, hi, f0, f1);
    int64_t w0 = 8 * c->wlo[ax], w1 = 8 * c->whi[ax] + 7;
    if (*f0 < w0) *f0 = w0;
    if (*f1 > w1) *f1 = w1;
    if (*f0 < 0) *f0 = 0;
    if (*f1 > N8 - 1) *f1 = N8 - 1;
    return *f0 <= *f1;
}

int orc_density_fibers(orc_ctx* c, const float* seg, const float* radii, uint64_t S) {
    int rc = density_prepare(c);
    if (rc) return rc;
    for (uint64_t p = 0; p < S; p++) {
        float a[3], b[3];
        for (int ax = 0; ax < 3; ax++) {
            a[ax] = 8.0f * grid_coord(&c->g, ax, seg[6 * p + ax]);
            b[ax] = 8.0f * grid_coord(&c->g, ax, seg[6 * p + 3 + ax]);
        }
        float rg = 8.0f * grid_len(&c->g, radii[p]);
        int64_t f0[3], f1[3];
        int ok = 1;
        for (int ax = 0; ax < 3; ax++) {
            float lo = fminf_(a[ax], b[ax]) - rg, hi = fmaxf_(a[ax], b[ax]) + rg;
            if (!fine_range(c, ax, lo, hi, &f0[ax], &f1[ax])) ok = 0;
        }
        if (!ok) continue;
        if ((f1[0] - f0[0] + 1) * (f1[1] - f0[1] + 1) * (f1[2] - f0[2] + 1) > (1ll << 26)) return ORC_ERR_ARG;
        fiber_t f;
        fiber_setup(&f, a, b, rg);
        for (int64_t z = f0[2]; z <= f1[2]; z++)
            for (int64_t y = f0[1]; y <= f1[1]; y++)
                for (int64_t x = f0[0]; x <= f1[0]; x++) {
                    float ell;
                    if (fiber_eval(&f, x, y, z, &ell)) density_set(c, x, y, z);
                }
    }
    return ORC_OK;
}

int orc_density_triangles(orc_ctx* c, const float* tri, uint64_t T) {
    int rc = density_prepare(c);
    if (rc) return rc;
    for (uint64_t t = 0; t < T; t++) {
        float g[9];
        for (int q = 0; q < 9; q++) g[q] = 8.0f * grid_coord(&c->g, q % 3, tri[9 * t + q]);
        int64_t f0[3], f1[3];
        int ok = 1;
        for (int ax = 0; ax < 3; ax++) {
            float lo = fminf_(fminf_(g[ax], g[3 + ax]), g[6 + ax]);
            float hi = fmaxf_(fmaxf_(g[ax], g[3 + ax]), g[6 + ax]);
            if (!fine_range(c, ax, lo, hi, &f0[ax], &f1[ax])) ok = 0;
        }
        if (!ok) continue;
        if ((f1[0] - f0[0] + 1) * (f1[1] - f0[1] + 1) * (f1[2] - f0[2] + 1) > (1ll << 26)) return ORC_ERR_ARG;
        for (int64_t z = f0[2]; z <= f1[2]; z++)
            for (int64_t y = f0[1]; y <= f1[1]; y++)
                for (int64_t x = f0[0]; x <= f1[0]; x++)
                    if (tri_sat(g, x, y, z)) density_set(c, x, y, z);
    }
    return ORC_OK;
}

/* Masks of level l (direct from level 0: a level-0 sub-voxel at fine offset X inside a
 * level-l voxel lands in the level-l sub-voxel X >> l), occupancy = hits / 512 and
 * the coverage of the projections onto the YZ, XZ, XY planes / 64. */
int orc_density_level(const orc_ctx* c, int l, uint64_t* masks, float* occ, float* axis) {
    if (l < 0 || l > c->built || !c->dm0) return ORC_ERR_LEVEL;
    const level_t* L = &c->lv[l];
    uint64_t* m = (uint64_t*)calloc((L->n ? L->n : 1) * 8, sizeof(uint64_t));
    if (!m) return ORC_ERR_OOM;
    const level_t* L0 = &c->lv[0];
    for (uint64_t v = 0; v < L0->n; v++) {
        uint32_t i, j, k;
        orc_unmorton(L0->key[v], &i, &j, &k);
        int64_t pv = key_index(L, L0->key[v] >> (3 * l));
        if (pv < 0) continue;
        uint32_t span = 1u << l;
        for (int cz = 0; cz < 8; cz++)
            for (int cy = 0; cy < 8; cy++)
                for (int cx = 0; cx < 8; cx++) {
                    if (!((c->dm0[8 * v + cz] >> (cx + 8 * cy)) & 1ull)) continue;
                    uint32_t X = 8 * (i % span) + cx, Y = 8 * (j % span) + cy, Z = 8 * (k % span) + cz;
                    uint32_t A = X >> l, B = Y >> l, C = Z >> l;
                    m[8 * pv + C] |= 1ull << (A + 8 * B);
                }
    }
    for (uint64_t v = 0; v < L->n; v++) {
        const uint64_t* w = m + 8 * v;
        uint64_t xy = 0, hits = 0, xz = 0, yz = 0;
        for (int cz = 0; cz < 8; cz++) {
            xy |= w[cz];
            hits += (uint64_t)__builtin_popcountll(w[cz]);
            for (int cy = 0; cy < 8; cy++)
                for (int cx = 0; cx < 8; cx++)
                    if ((w[cz] >> (cx + 8 * cy)) & 1ull) {
                        xz |= 1ull << (cx + 8 * cz);
                        yz |= 1ull << (cy + 8 * cz);
                    }
        }
        if (masks) memcpy(masks + 8 * v, w, 64);
        if (occ) occ[v] = (float)hits / 512.0f;
        if (axis) {
            axis[3 * v + 0] = (float)__builtin_popcountll(yz) / 64.0f;
            axis[3 * v + 1] = (float)__builtin_popcountll(xz) / 64.0f;
            axis[3 * v + 2] = (float)__builtin_popcountll(xy) / 64.0f;
        }
    }
    free(m);
    return ORC_OK;
}

/* ------------------------------------------------------------------ §9 SGGX-H */

static void theta_table(float theta[32][3], float coef[32][6]) {
    const double PI_D = 3.14159265358979323846;
    const double ga = PI_D * (3.0 - sqrt(5.0));
    for (int k = 0; k < 32; k++) {
        double z = 1.0 - (k + 0.5) / 32.0;
        double rho = sqrt(1.0 - z * z);
        double phi = k * ga;
        theta[k][0] = (float)(rho * cos(phi));
        theta[k][1] = (float)(rho * sin(phi));
        theta[k][2] = (float)z;
        double x = theta[k][0], y = theta[k][1], zz = theta[k][2];
        coef[k][0] = (float)(x * x);
        coef[k][1] = (float)(y * y);
        coef[k][2] = (float)(zz * zz);
        coef[k][3] = (float)(2.0 * x * y);
        coef[k][4] = (float)(2.0 * x * zz);
        coef[k][5] = (float)(2.0 * y * zz);
    }
}

void orc_theta(float* theta, float* coef) {
    float t[32][3], c[32][6];
    theta_table(t, c);
    memcpy(theta, t, sizeof(t));
    memcpy(coef, c, sizeof(c));
}

/* sigma_k of one cluster from its accumulators (w, Mxx, Myy, Mzz, Mxy, Mxz, Myz) */
static void cluster_sigma(const i128 acc[7], const float coef[32][6], float sig[32]) {
    float wf = deq32(acc[0]);
    float S[6];
    for (int e = 0; e < 6; e++) S[e] = deq32(acc[1 + e]) / wf;
    for (int k = 0; k < 32; k++) {
        float q = coef[k][0] * S[0];
        for (int e = 1; e < 6; e++) q = q + coef[k][e] * S[e];
        sig[k] = sqrtf(fmaxf_(q, 0.0f));
    }
}

static float sigma_dist(const float si[32], const float sj[32]) {
    float s[32];
    for (int k = 0; k < 32; k++) s[k] = fabsf(si[k] - sj[k]);
    for (int h = 16; h >= 1; h >>= 1)
        for (int l = 0; l < h; l++) s[l] = s[l] + s[l + h];
    return s[0];
}

/* SGGX-H on n clusters (in order), down to K. Clusters are [n][7] i128, modified in
 * place; returns the number kept. P:383-387: D_{L-1} = (D_L \ {S_i,S_j}) U S_n. */
static int sggxh(i128 (*cl)[7], int n, int K, const float coef[32][6]) {
    float sig[8 * MAX_K][32];
    while (n > K) {
        for (int c = 0; c < n; c++) cluster_sigma(cl[c], coef, sig[c]);
        int bi = 0, bj = 1;
        float best = 0.0f;
        int have = 0;
        for (int i = 0; i < n; i++)
            for (int j = i + 1; j < n; j++) {
                float d = sigma_dist(sig[i], sig[j]);
                if (!have || d < best) { best = d; bi = i; bj = j; have = 1; }
            }
        for (int e = 0; e < 7; e++) cl[bi][e] += cl[bj][e];
        for (int c = bj; c + 1 < n; c++) memcpy(cl[c], cl[c + 1], sizeof(cl[c]));
        n--;
    }
    return n;
}

/* Unit entry: n clusters of int64 accumulators -> out [K][7]; returns ncl. */
int orc_sggxh(int n, const int64_t* acc, int K, int64_t* out) {
    if (n < 0 || n > 8 * MAX_K || K < 1 || K > MAX_K) return ORC_ERR_ARG;
    float theta[32][3], coef[32][6];
    theta_table(theta, coef);
    i128 cl[8 * MAX_K][7];
    int m = 0;
    for (int c = 0; c < n; c++) {
        if (acc[7 * c] == 0) continue; /* w = 0 clusters are dropped */
        for (int e = 0; e < 7; e++) cl[m][e] = acc[7 * c + e];
        m++;
    }
    if (m > K) m = sggxh(cl, m, K, coef);
    for (int c = 0; c < m; c++)
        for (int e = 0; e < 7; e++) {
            if (!fits64(cl[c][e])) return ORC_ERR_OVERFLOW;
            out[7 * c + e] = (int64_t)cl[c][e];
        }
    return m;
}

void orc_sigma(const int64_t acc[7], float sig[32]) {
    float theta[32][3], coef[32][6];
    theta_table(theta, coef);
    i128 a[7];
    for (int e = 0; e < 7; e++) a[e] = acc[e];
    cluster_sigma(a, coef, sig);
}

float orc_distance(const int64_t a[7], const int64_t b[7]) {
    float sa[32], sb[32];
    orc_sigma(a, sa);
    orc_sigma(b, sb);
    return sigma_dist(sa, sb);
}

/* ------------------------------------------------------------------ §10 histogram distance */
/* distance_mode = hist: the paper's own distance, a Wasserstein
 * distance between 5x5x5 histograms of N whole-sphere samples of each SGGX (P:383-389,
 * P:341), taken as the sliced W1 over the 32 slices of §9 in exact
 * integer arithmetic. Merges stay exact moment sums (D15); a merged cluster's histogram
 * is drawn afresh from its S. */

/* sample table: N spherical-Fibonacci points over the whole sphere, fp64 -> fp32 */
static void sample_table(int N, float (*u)[3]) {
    const double PI_D = 3.14159265358979323846;
    const double ga = PI_D * (3.0 - sqrt(5.0));
    for (int s = 0; s < N; s++) {
        double z = 1.0 - (2.0 * s + 1.0) / N;
        double rho = sqrt(1.0 - z * z);
        double phi = s * ga;
        u[s][0] = (float)(rho * cos(phi));
        u[s][1] = (float)(rho * sin(phi));
        u[s][2] = (float)z;
    }
}

/* slice tables: fixed-point projections P[k][b] of the bin centres, bins sorted by
 * (P, b) and the gaps between consecutive sorted projections */
static void sw_tables(const float theta[32][3], uint8_t perm[32][HIST_BINS], int64_t gap[32][HIST_BINS - 1]) {
    for (int k = 0; k < 32; k++) {
        int64_t P[HIST_BINS];
        int idx[HIST_BINS];
        for (int b = 0; b < HIST_BINS; b++) {
            int b0 = b % 5, b1 = (b / 5) % 5, b2 = b / 25;
            double x = (double)theta[k][0] * (2 * b0 - 4) + (double)theta[k][1] * (2 * b1 - 4);
            x = x + (double)theta[k][2] * (2 * b2 - 4);
            P[b] = llrint(x * 65536.0);
            idx[b] = b;
        }
        for (int a = 1; a < HIST_BINS; a++) { /* insertion sort by (P, b) */
            int v = idx[a], m = a;
            while (m > 0 && (P[idx[m - 1]] > P[v] || (P[idx[m - 1]] == P[v] && idx[m - 1] > v))) {
                idx[m] = idx[m - 1];
                m--;
            }
            idx[m] = v;
        }
        for (int r = 0; r < HIST_BINS; r++) perm[k][r] = (uint8_t)idx[r];
        for (int r = 0; r + 1 < HIST_BINS; r++) gap[k][r] = P[idx[r + 1]] - P[idx[r]];
    }
}

/* histogram of one cluster: Cholesky factor L of S = M / w (L L^T = S), samples
 * normalize(L u_s), binned per component by floor((d + 1) * 2.5) clamped to [0, 4] */
static void cluster_hist(const i128 acc[7], const float (*u)[3], int N, uint16_t H[HIST_BINS]) {
    float wf = deq32(acc[0]);
    float S[6];
    for (int e = 0; e < 6; e++) S[e] = deq32(acc[1 + e]) / wf;
    float L00 = sqrtf(fmaxf_(S[0], 0.0f));
    float L10 = L00 > 0.0f ? S[3] / L00 : 0.0f;
    float L20 = L00 > 0.0f ? S[4] / L00 : 0.0f;
    float t = S[1] - L10 * L10;
    float L11 = sqrtf(fmaxf_(t, 0.0f));
    float L21 = L11 > 0.0f ? (S[5] - L20 * L10) / L11 : 0.0f;
    t = (S[2] - L20 * L20) - L21 * L21;
    float L22 = sqrtf(fmaxf_(t, 0.0f));
    memset(H, 0, sizeof(uint16_t) * HIST_BINS);
    for (int s = 0; s < N; s++) {
        float v0 = L00 * u[s][0];
        float v1 = L10 * u[s][0] + L11 * u[s][1];
        float v2 = (L20 * u[s][0] + L21 * u[s][1]) + L22 * u[s][2];
        float n2 = (v0 * v0 + v1 * v1) + v2 * v2;
        int b[3] = {2, 2, 2};
        if (n2 > 0.0f) {
            float r = sqrtf(n2);
            float inv = 1.0f / r;
            float d[3] = {v0 * inv, v1 * inv, v2 * inv};
            for (int c = 0; c < 3; c++) {
                int bi = (int)floorf((d[c] + 1.0f) * 2.5f);
                b[c] = bi < 0 ? 0 : (bi > 4 ? 4 : bi);
            }
        }
        H[b[0] + 5 * b[1] + 25 * b[2]]++;
    }
}

/* d_hist = sum over slices k of sum_r |C_r| * gap[k][r], C_r the running count difference */
static int64_t hist_dist(const uint16_t* Hi, const uint16_t* Hj, const uint8_t perm[32][HIST_BINS],
                         const int64_t gap[32][HIST_BINS - 1]) {
    int64_t d = 0;
    for (int k = 0; k < 32; k++) {
        int64_t C = 0, W = 0;
        for (int r = 0; r + 1 < HIST_BINS; r++) {
            C += (int64_t)Hi[perm[k][r]] - (int64_t)Hj[perm[k][r]];
            W += (C < 0 ? -C : C) * gap[k][r];
        }
        d += W;
    }
    return d;
}


static int hist_tables_init(hist_tables_t* T, int N) {
    if (N < HIST_NMIN || N > HIST_NMAX) return ORC_ERR_ARG;
    float theta[32][3], coef[32][6];
    theta_table(theta, coef);
    T->N = N;
    T->u = (float(*)[3])malloc(sizeof(float) * 3 * N);
    if (!T->u) return ORC_ERR_OOM;
    sample_table(N, T->u);
    sw_tables(theta, T->perm, T->gap);
    return ORC_OK;
}

/* SGGX-H (§9) with d_hist; histograms are kept per cluster and redrawn for a merged one */
static int sggxh_hist(i128 (*cl)[7], int n, int K, const hist_tables_t* T) {
    uint16_t H[8 * MAX_K][HIST_BINS];
    for (int c = 0; c < n; c++) cluster_hist(cl[c], (const float(*)[3])T->u, T->N, H[c]);
    while (n > K) {
        int bi = 0, bj = 1, have = 0;
        int64_t best = 0;
        for (int i = 0; i < n; i++)
            for (int j = i + 1; j < n; j++) {
                int64_t d = hist_dist(H[i], H[j], T->perm, T->gap);
                if (!have || d < best) { best = d; bi = i; bj = j; have = 1; }
            }
        for (int e = 0; e < 7; e++) cl[bi][e] += cl[bj][e];
        cluster_hist(cl[bi], (const float(*)[3])T->u, T->N, H[bi]);
        for (int c = bj; c + 1 < n; c++) {
            memcpy(cl[c], cl[c + 1], sizeof(cl[c]));
            memcpy(H[c], H[c + 1], sizeof(H[c]));
        }
        n--;
    }
    return n;
}

void orc_sample_table(int N, float* out) { sample_table(N, (float(*)[3])out); }

void orc_sw_tables(uint8_t* perm, int64_t* gap) {
    float theta[32][3], coef[32][6];
    theta_table(theta, coef);
    sw_tables(theta, (uint8_t(*)[HIST_BINS])perm, (int64_t(*)[HIST_BINS - 1])gap);
}

int orc_hist(const int64_t acc[7], int N, uint16_t* H) {
    hist_tables_t T;
    int rc = hist_tables_init(&T, N);
    if (rc != ORC_OK) return rc;
    i128 a[7];
    for (int e = 0; e < 7; e++) a[e] = acc[e];
    cluster_hist(a, (const float(*)[3])T.u, N, H);
    free(T.u);
    return ORC_OK;
}

int64_t orc_hist_distance(const uint16_t* Hi, const uint16_t* Hj) {
    float theta[32][3], coef[32][6];
    uint8_t perm[32][HIST_BINS];
    int64_t gap[32][HIST_BINS - 1];
    theta_table(theta, coef);
    sw_tables(theta, perm, gap);
    return hist_dist(Hi, Hj, perm, gap);
}

int orc_sggxh_hist(int n, const int64_t* acc, int K, int N, int64_t* out) {
    if (n < 0 || n > 8 * MAX_K || K < 1 || K > MAX_K) return ORC_ERR_ARG;
    hist_tables_t T;
    int rc = hist_tables_init(&T, N);
    if (rc != ORC_OK) return rc;
    i128 cl[8 * MAX_K][7];
    int m = 0;
    for (int c = 0; c < n; c++) {
        if (acc[7 * c] == 0) continue;
        for (int e = 0; e < 7; e++) cl[m][e] = acc[7 * c + e];
        m++;
    }
    if (m > K) m = sggxh_hist(cl, m, K, &T);
    free(T.u);
    for (int c = 0; c < m; c++)
        for (int e = 0; e < 7; e++) {
            if (!fits64(cl[c][e])) return ORC_ERR_OVERFLOW;
            out[7 * c + e] = (int64_t)cl[c][e];
        }
    return m;
}

/* ------------------------------------------------------------------ §11 compact form */
/* SGGX finalisation: eigenvalues by pinned cyclic Jacobi, degenerate
 * jitter in moment form, normalisation to max projected area 1, the 6-byte compact
 * form of Eq. compact-sggx. */
static void jacobi3(const float S[6], float lam[3]) {
    float a[3][3] = {{S[0], S[3], S[4]}, {S[3], S[1], S[5]}, {S[4], S[5], S[2]}};
    static const int PQ[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    for (int sweep = 0; sweep < 6; sweep++) {
        int rotated = 0;
        for (int m = 0; m < 3; m++) {
            int p = PQ[m][0], q = PQ[m][1], r = 3 - p - q;
            float apq = a[p][q];
            /* negligible off-diagonal (relative 2^-24 of the diagonal): no rotation */
            if (!(fabsf(apq) * 16777216.0f > fabsf(a[p][p]) + fabsf(a[q][q]))) continue;
            rotated = 1;
            float th = (a[q][q] - a[p][p]) / (2.0f * apq);
            float t = 1.0f / (fabsf(th) + sqrtf(th * th + 1.0f));
            if (th < 0.0f) t = -t;
            float c = 1.0f / sqrtf(t * t + 1.0f);
            float sn = t * c;
            a[p][p] = a[p][p] - t * apq;
            a[q][q] = a[q][q] + t * apq;
            a[p][q] = a[q][p] = 0.0f;
            float arp = a[r][p], arq = a[r][q];
            a[r][p] = a[p][r] = c * arp - sn * arq;
            a[r][q] = a[q][r] = sn * arp + c * arq;
        }
        if (!rotated) break;   /* a sweep without rotation: converged */
    }
    lam[0] = a[0][0];
    lam[1] = a[1][1];
    lam[2] = a[2][2];
}

static uint8_t byte_sigma(float x) {
    int b = (int)floorf(x * 255.0f + 0.5f);
    return (uint8_t)(b > 255 ? 255 : (b < 0 ? 0 : b));
}
static uint8_t byte_r(float r) {
    int b = (int)floorf((r + 1.0f) * 127.5f + 0.5f);
    return (uint8_t)(b > 255 ? 255 : (b < 0 ? 0 : b));
}
static float corr(float sxy, float sxx, float syy) {
    float p = sxx * syy;
    float r = p > 0.0f ? sxy / sqrtf(p) : 0.0f;
    return r > 1.0f ? 1.0f : (r < -1.0f ? -1.0f : r);
}

/* §11 up to the normalised matrix: Sn [6]; returns 1 iff jittered, -1 if there is no SGGX
 * (w = 0 or max eigenvalue <= 0; Sn zero) */
static int finalize6(const i128 acc[7], float Sn[6]) {
    for (int e = 0; e < 6; e++) Sn[e] = 0.0f;
    if (acc[0] == 0) return -1;
    float wf = deq32(acc[0]);
    float S[6];
    for (int e = 0; e < 6; e++) S[e] = deq32(acc[1 + e]) / wf;
    float tr = (S[0] + S[1]) + S[2];
    float lam[3];
    jacobi3(S, lam);
    float lmax = lam[0], lmin = lam[0];
    for (int a = 1; a < 3; a++) {
        if (lam[a] > lmax) lmax = lam[a];
        if (lam[a] < lmin) lmin = lam[a];
    }
    int jit = lmin < 1e-4f * lmax;
    if (jit) {
        const float C1 = 0.9999f, C2 = (float)(1e-4 / 3.0);
        for (int e = 0; e < 6; e++) S[e] = e < 3 ? C1 * S[e] + C2 * tr : C1 * S[e];
        lmax = C1 * lmax + C2 * tr;
    }
    if (!(lmax > 0.0f)) return -1;
    float inv = 1.0f / lmax;
    for (int e = 0; e < 6; e++) Sn[e] = S[e] * inv;
    return jit;
}

/* returns 1 iff the record was jittered */
static int encode6(const i128 acc[7], uint8_t out[6]) {
    static const uint8_t ZERO[6] = {0, 0, 0, 128, 128, 128};
    memcpy(out, ZERO, 6);
    float Sn[6];
    int jit = finalize6(acc, Sn);
    if (jit < 0) return 0;
    out[0] = byte_sigma(sqrtf(fmaxf_(Sn[0], 0.0f)));
    out[1] = byte_sigma(sqrtf(fmaxf_(Sn[1], 0.0f)));
    out[2] = byte_sigma(sqrtf(fmaxf_(Sn[2], 0.0f)));
    out[3] = byte_r(corr(Sn[3], Sn[0], Sn[1]));
    out[4] = byte_r(corr(Sn[4], Sn[0], Sn[2]));
    out[5] = byte_r(corr(Sn[5], Sn[1], Sn[2]));
    return jit;
}

int orc_finalize(const int64_t acc7[7], float Sn[6]) {
    i128 a[7];
    for (int e = 0; e < 7; e++) a[e] = acc7[e];
    return finalize6(a, Sn);
}

void orc_jacobi(const float S[6], float lam[3]) { jacobi3(S, lam); }

/* n records of int64 (w, M6) -> out [n][6]; jit [n] (nullable) */
void orc_encode(uint64_t n, const int64_t* acc, uint8_t* out, uint8_t* jit) {
    for (uint64_t x = 0; x < n; x++) {
        i128 a[7];
        for (int e = 0; e < 7; e++) a[e] = acc[7 * x + e];
        int j = encode6(a, out + 6 * x);
        if (jit) jit[x] = (uint8_t)j;
    }
}

static int cmp_rec(const void* x, const void* y) {
    uint64_t a = ((const rec_t*)x)->key, b = ((const rec_t*)y)->key;
    return a < b ? -1 : a > b;
}

/* Leaf (§8, §9 level 0) then levels 1..levels (§9). */
static int build_up(orc_ctx* c, int levels);

int orc_build(orc_ctx* c, int levels) {
    if (levels < 0 || levels > c->logN) return ORC_ERR_LEVEL;
    free_levels(c);
    const int K = c->K;
    /* level 0: sort records by key and sum each run exactly */
    qsort(c->recs, c->nrec, sizeof(rec_t), cmp_rec);
    uint64_t V = 0;
    for (size_t r = 0; r < c->nrec; r++)
        if (r == 0 || c->recs[r].key != c->recs[r - 1].key) V++;
    level_t* L0 = &c->lv[0];
    L0->n = V;
    L0->key = (uint64_t*)malloc(sizeof(uint64_t) * (V ? V : 1));
    L0->acc = (i128*)calloc((V ? V : 1) * 7, sizeof(i128));
    L0->ncl = (uint8_t*)calloc(V ? V : 1, 1);
    L0->cl = (i128*)calloc((V ? V : 1) * K * 7, sizeof(i128));
    if (!L0->key || !L0->acc || !L0->ncl || !L0->cl) return ORC_ERR_OOM;
    int64_t v = -1;
    for (size_t r = 0; r < c->nrec; r++) {
        if (r == 0 || c->recs[r].key != c->recs[r - 1].key) { v++; L0->key[v] = c->recs[r].key; }
        for (int e = 0; e < 7; e++) L0->acc[7 * v + e] += c->recs[r].q[e];
    }
    for (uint64_t x = 0; x < V; x++) {
        for (int e = 0; e < 7; e++)
            if (!fits64(L0->acc[7 * x + e])) return ORC_ERR_OVERFLOW;
        if (L0->acc[7 * x] > 0) {
            L0->ncl[x] = 1;
            for (int e = 0; e < 7; e++) L0->cl[(size_t)x * K * 7 + e] = L0->acc[7 * x + e];
        }
    }
    c->built = 0;
    return build_up(c, levels);
}

/* Levels c->built + 1 .. levels from level c->built (P:364 sums, P:376-387 SGGX-H). */
static int build_up(orc_ctx* c, int levels) {
    const int K = c->K;
    float theta[32][3], coef[32][6];
    theta_table(theta, coef);
    for (int l = c->built + 1; l <= levels; l++) {
        level_t* Cc = &c->lv[l - 1];
        level_t* P = &c->lv[l];
        uint64_t nP = 0;
        for (uint64_t x = 0; x < Cc->n; x++)
            if (x == 0 || (Cc->key[x] >> 3) != (Cc->key[x - 1] >> 3)) nP++;
        P->n = nP;
        P->key = (uint64_t*)malloc(sizeof(uint64_t) * (nP ? nP : 1));
        P->acc = (i128*)calloc((nP ? nP : 1) * 7, sizeof(i128));
        P->ncl = (uint8_t*)calloc(nP ? nP : 1, 1);
        P->cl = (i128*)calloc((nP ? nP : 1) * K * 7, sizeof(i128));
        if (!P->key || !P->acc || !P->ncl || !P->cl) return ORC_ERR_OOM;
        uint64_t x = 0, p = 0;
        while (x < Cc->n) {
            uint64_t pk = Cc->key[x] >> 3;
            i128 list[8 * MAX_K][7];
            int n = 0;
            P->key[p] = pk;
            while (x < Cc->n && (Cc->key[x] >> 3) == pk) {
                for (int e = 0; e < 7; e++) P->acc[7 * p + e] += Cc->acc[7 * x + e];
                for (int q = 0; q < Cc->ncl[x]; q++) {
                    const i128* src = &Cc->cl[((size_t)x * K + q) * 7];
                    if (src[0] == 0) continue;
                    for (int e = 0; e < 7; e++) list[n][e] = src[e];
                    n++;
                }
                x++;
            }
            if (n > K) n = c->mode == 1 ? sggxh_hist(list, n, K, c->ht) : sggxh(list, n, K, coef);
            P->ncl[p] = (uint8_t)n;
            for (int q = 0; q < n; q++)
                for (int e = 0; e < 7; e++) {
                    if (!fits64(list[q][e])) return ORC_ERR_OVERFLOW;
                    P->cl[((size_t)p * K + q) * 7 + e] = list[q][e];
                }
            for (int e = 0; e < 7; e++)
                if (!fits64(P->acc[7 * p + e])) return ORC_ERR_OVERFLOW;
            p++;
        }
        c->built = l;
    }
    return ORC_OK;
}

/* Test infrastructure: start the pyramid from given records of level l0 (sorted keys, exact
 * accumulators acc [n][7], lobe counts ncl [n] and lobe accumulators clacc [n][K][7]; for
 * l0 = 0 ncl / clacc are ignored and derived from acc as in orc_build) and build levels
 * l0 + 1 .. levels with the same code as orc_build. Lets a test check the upper levels of a
 * workload too large for the oracle's voxelization against the GPU's records of level l0. */
int orc_build_from(orc_ctx* c, int l0, uint64_t n, const uint64_t* key, const int64_t* acc, const uint8_t* ncl,
                   const int64_t* clacc, int levels) {
    if (l0 < 0 || l0 > levels || levels > c->logN) return ORC_ERR_LEVEL;
    free_levels(c);
    const int K = c->K;
    level_t* L = &c->lv[l0];
    L->n = n;
    L->key = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    L->acc = (i128*)calloc((n ? n : 1) * 7, sizeof(i128));
    L->ncl = (uint8_t*)calloc(n ? n : 1, 1);
    L->cl = (i128*)calloc((n ? n : 1) * K * 7, sizeof(i128));
    if (!L->key || !L->acc || !L->ncl || !L->cl) return ORC_ERR_OOM;
    for (uint64_t x = 0; x < n; x++) {
        if (x > 0 && key[x] <= key[x - 1]) return ORC_ERR_ARG;
        L->key[x] = key[x];
        for (int e = 0; e < 7; e++) L->acc[7 * x + e] = acc[7 * x + e];
        if (l0 == 0) {
            if (acc[7 * x] > 0) {
                L->ncl[x] = 1;
                for (int e = 0; e < 7; e++) L->cl[(size_t)x * K * 7 + e] = acc[7 * x + e];
            }
        } else {
            if (ncl[x] > K) return ORC_ERR_ARG;
            L->ncl[x] = ncl[x];
            for (int q = 0; q < ncl[x]; q++)
                for (int e = 0; e < 7; e++) L->cl[((size_t)x * K + q) * 7 + e] = clacc[((size_t)x * K + q) * 7 + e];
        }
    }
    c->built = l0;
    return build_up(c, levels);
}

uint64_t orc_level_size(const orc_ctx* c, int l) {
    if (l < 0 || l > c->built) return 0;
    return c->lv[l].n;
}

/* Copy level l out: keys, int64 accumulators [n][7], fp32 mass/m6, ncl, cluster
 * accumulators [n][K][7] and fp32 clusters [n][K][7] (unused slots zero). */
int orc_level_copy(const orc_ctx* c, int l, uint64_t* key, int64_t* acc, float* mass, float* m6,
                   uint8_t* ncl, int64_t* clacc, float* cl) {
    if (l < 0 || l > c->built) return ORC_ERR_LEVEL;
    const level_t* L = &c->lv[l];
    const int K = c->K;
    for (uint64_t x = 0; x < L->n; x++) {
        if (key) key[x] = L->key[x];
        for (int e = 0; e < 7; e++) {
            i128 a = L->acc[7 * x + e];
            if (acc) acc[7 * x + e] = (int64_t)a;
            if (e == 0) { if (mass) mass[x] = deq32(a); }
            else if (m6) m6[6 * x + e - 1] = deq32(a);
        }
        if (ncl) ncl[x] = L->ncl[x];
        for (int q = 0; q < K; q++)
            for (int e = 0; e < 7; e++) {
                i128 a = L->cl[((size_t)x * K + q) * 7 + e];
                if (clacc) clacc[((size_t)x * K + q) * 7 + e] = (int64_t)a;
                if (cl) cl[((size_t)x * K + q) * 7 + e] = q < L->ncl[x] ? deq32(a) : 0.0f;
            }
    }
    return ORC_OK;
}
