// k_fiber.cu -- fiber segments: cull/bin (k_fiber_bound) and capsule-box overlap + emit
// (k_fiber_emit). docs/PREDICATES.md §1, §3, §4, §5 (north star: fiber-capsule-box test
// emitting (Morton key, contribution) pairs; P:190-198 block test as a conservative cull;
// P:224-228 t-uniform curve sampling whose continuous limit is the ball-touch length).
#include "vox_internal.cuh"

namespace vox {

VOX_DEBUG_TU(fiber)

struct SegGeom {
    float a[3], b[3], rg;
    bool culled;
    bool too_many;
    int64_t u0[3], u1[3];   // unclamped candidate range (§3)
    int64_t e0[3], e1[3];   // emission range (clamped to the grid)
};

// §1 + §3 for one segment (shared by the bound and emit kernels).
__device__ __forceinline__ void seg_geom(const GridXf& g, const float* s, float r, SegGeom& G) {
    for (int ax = 0; ax < 3; ax++) {
        G.a[ax] = to_grid(g, ax, s[ax]);
        G.b[ax] = to_grid(g, ax, s[3 + ax]);
    }
    G.rg = to_grid_len(g, r);
    G.culled = false;
    G.too_many = false;
    const float Nhi = g.Nf + 1.0f;
    for (int ax = 0; ax < 3; ax++) {
        float lo = pmin(G.a[ax], G.b[ax]) - G.rg;
        float hi = pmax(G.a[ax], G.b[ax]) + G.rg;
        if (!(hi >= -1.0f) || !(lo <= Nhi)) { G.culled = true; return; }
        if (hi - lo > 16777216.0f) { G.too_many = true; G.culled = true; return; }
        G.u0[ax] = (int64_t)ceilf(lo) - 1;
        G.u1[ax] = (int64_t)floorf(hi);
        G.e0[ax] = G.u0[ax] < 0 ? 0 : G.u0[ax];
        G.e1[ax] = G.u1[ax] > g.N - 1 ? g.N - 1 : G.u1[ax];
        if (G.e0[ax] > G.e1[ax]) G.culled = true;
    }
    if (!G.culled) {
        uint64_t n = (uint64_t)(G.u1[0] - G.u0[0] + 1) * (uint64_t)(G.u1[1] - G.u0[1] + 1) *
                     (uint64_t)(G.u1[2] - G.u0[2] + 1);
        if (n > (1ull << 24)) { G.too_many = true; G.culled = true; }
    }
}

// Adds the clamped candidate count of box [e0,e1] to each top cell it overlaps (cell edge
// = 2^s voxels). Used for capacity (exact upper bound on pairs per cell) and sharding.
__device__ __forceinline__ void add_cells(const int64_t* e0, const int64_t* e1, int s,
                                          unsigned long long* cellW) {
    const int64_t c0x = e0[0] >> s, c1x = e1[0] >> s;
    const int64_t c0y = e0[1] >> s, c1y = e1[1] >> s;
    const int64_t c0z = e0[2] >> s, c1z = e1[2] >> s;
    for (int64_t cz = c0z; cz <= c1z; cz++) {
        int64_t nz = min(e1[2], ((cz + 1) << s) - 1) - max(e0[2], cz << s) + 1;
        for (int64_t cy = c0y; cy <= c1y; cy++) {
            int64_t ny = min(e1[1], ((cy + 1) << s) - 1) - max(e0[1], cy << s) + 1;
            for (int64_t cx = c0x; cx <= c1x; cx++) {
                int64_t nx = min(e1[0], ((cx + 1) << s) - 1) - max(e0[0], cx << s) + 1;
                atomicAdd(&cellW[morton3((uint32_t)cx, (uint32_t)cy, (uint32_t)cz)],
                          (unsigned long long)(nx * ny * nz));
            }
        }
    }
}

__global__ void k_fiber_bound(const float* __restrict__ seg, const float* __restrict__ rad, uint64_t S,
                              GridXf g, int cell_shift, unsigned long long* __restrict__ cellW,
                              unsigned* __restrict__ flags) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < S;
         p += (uint64_t)gridDim.x * blockDim.x) {
        float s[6];
        for (int q = 0; q < 6; q++) s[q] = seg[6 * p + q];
        const float r = rad[p];
        bool bad = false;
        for (int q = 0; q < 6; q++) bad |= !isfinite(s[q]);
        bad |= !isfinite(r);
        if (bad) { atomicOr(flags, VOX_EFLAG_NONFINITE); continue; }
        if (r < 0.0f) { atomicOr(flags, VOX_EFLAG_NEG_RADIUS); continue; }
        SegGeom G;
        seg_geom(g, s, r, G);
        if (G.too_many) { atomicOr(flags, VOX_EFLAG_TOO_MANY_CAND); continue; }
        if (G.culled) continue;
        add_cells(G.e0, G.e1, cell_shift, cellW);
    }
}

// ---------------------------------------------------------------- §4 capsule-box predicate

struct Fib {
    float a[3], w[3], iota[3];
    float r2, len;
    unsigned moving;   // bit ax set iff w_ax > 0
};

// Sorting network for 6 values (ascending); values outside (0,1) were replaced by 1.
__device__ __forceinline__ void cswap(float& x, float& y) {
    float lo = pmin(x, y), hi = pmax(x, y);
    x = lo; y = hi;
}

// Returns true iff voxel (i,j,k) is a key; ell = l_r. Pinned sequence of PREDICATES §4.
__device__ __forceinline__ bool fiber_key(const Fib& f, int64_t i, int64_t j, int64_t k, float& ell) {
    const float lo[3] = {(float)i, (float)j, (float)k};
    const float hi[3] = {(float)(i + 1), (float)(j + 1), (float)(k + 1)};
    float u[3], v[3], Wu[3], Wuu[3], Wv[3], Wvv[3];
    float C0 = 0.0f;
    float bp[6];
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        if (f.moving & (1u << ax)) {
            float t1 = (lo[ax] - f.a[ax]) * f.iota[ax];
            float t2 = (hi[ax] - f.a[ax]) * f.iota[ax];
            u[ax] = pmin(t1, t2);
            v[ax] = pmax(t1, t2);
            Wu[ax] = f.w[ax] * u[ax];
            Wuu[ax] = Wu[ax] * u[ax];
            Wv[ax] = f.w[ax] * v[ax];
            Wvv[ax] = Wv[ax] * v[ax];
            // breakpoints outside (0, 1) become 1.0: sorted behind the interior ones, so the
            // piece ends are H_p = bp[p] for every piece p <= m (the last one ends at 1)
            bp[2 * ax] = (u[ax] > 0.0f && u[ax] < 1.0f) ? u[ax] : 1.0f;
            bp[2 * ax + 1] = (v[ax] > 0.0f && v[ax] < 1.0f) ? v[ax] : 1.0f;
        } else {
            // a fixed axis takes the u >= H branch below with w = Wu = Wuu = 0: adding +0 leaves
            // A, B, C bit-identical to skipping the axis (none of them is ever -0), so the piece
            // loop needs no per-axis moving test
            u[ax] = v[ax] = 2.0f;
            Wu[ax] = Wuu[ax] = Wv[ax] = Wvv[ax] = 0.0f;
            float c = 0.0f;
            if (f.a[ax] < lo[ax]) c = lo[ax] - f.a[ax];
            else if (f.a[ax] > hi[ax]) c = f.a[ax] - hi[ax];
            C0 = C0 + c * c;
            bp[2 * ax] = bp[2 * ax + 1] = 1.0f;
        }
    }
    // optimal 12-comparator network for 6 inputs
    cswap(bp[1], bp[2]); cswap(bp[4], bp[5]); cswap(bp[0], bp[2]); cswap(bp[3], bp[5]);
    cswap(bp[0], bp[1]); cswap(bp[3], bp[4]); cswap(bp[1], bp[4]); cswap(bp[0], bp[3]);
    cswap(bp[2], bp[5]); cswap(bp[1], bp[3]); cswap(bp[2], bp[4]); cswap(bp[2], bp[3]);
    int m = 0;
#pragma unroll
    for (int q = 0; q < 6; q++) m += bp[q] < 1.0f;   // interior breakpoints

    bool found = false;
    float ta = 0.0f, tb = 0.0f;
#pragma unroll
    for (int p = 0; p < 7; p++) {
        if (p > m) break;
        const float L = p == 0 ? 0.0f : bp[p - 1];
        const float H = p < 6 ? bp[p] : 1.0f;   // compile-time p: bp[m] = 1 when m < 6
        float A = 0.0f, B = 0.0f, C = C0;
#pragma unroll
        for (int ax = 0; ax < 3; ax++) {
            if (u[ax] >= H) { A = A + f.w[ax]; B = B + Wu[ax]; C = C + Wuu[ax]; }
            else if (v[ax] <= L) { A = A + f.w[ax]; B = B + Wv[ax]; C = C + Wvv[ax]; }
        }
        float lo_m, hi_m;
        if (A == 0.0f) {
            if (!(C <= f.r2)) continue;
            lo_m = L; hi_m = H;
        } else {
            float Cr = C - f.r2;
            float D = B * B - A * Cr;
            if (D < 0.0f) continue;
            float s = sqrtf(D);
            float t1 = (B - s) / A;
            float t2 = (B + s) / A;
            lo_m = pmax(t1, L);
            hi_m = pmin(t2, H);
            if (!(lo_m <= hi_m)) continue;
        }
        // pieces are ordered and lo >= L, hi <= H inside a piece, so over the feasible pieces
        // min lo is the first one's lo and max hi the last one's hi (the pinned pmin / pmax
        // would return exactly these values)
        if (!found) ta = lo_m;
        tb = hi_m;
        found = true;
    }
    if (!found) return false;
    ell = f.len * (tb - ta);
    return true;
}

// GPU-only conservative early reject (not part of the pinned definition): the voxel cannot be
// a key when its centre is farther than r + sqrt(3)/2 + 0.05 voxel from the segment, because
// every point of the box lies within sqrt(3)/2 of the centre and the pinned fp32 predicate
// deviates from the exact one by orders of magnitude less than 0.05 voxel. Parity tests
// compare the emitted key sets with the oracle, which has no such shortcut.
__device__ __forceinline__ bool far_from_capsule(const float* a, const float* d, float iww, float thr2, int64_t i,
                                                 int64_t j, int64_t k) {
    // conservative geometry (not the pinned predicate): fused multiply-adds are fine here
    const float e0 = ((float)i + 0.5f) - a[0], e1 = ((float)j + 0.5f) - a[1], e2 = ((float)k + 0.5f) - a[2];
    float t = __fmaf_rn(e2, d[2], __fmaf_rn(e1, d[1], e0 * d[0])) * iww;   // iww = 1 / |d|^2 (0 for a sphere)
    t = fminf(fmaxf(t, 0.0f), 1.0f);
    const float q0 = __fmaf_rn(-t, d[0], e0), q1 = __fmaf_rn(-t, d[1], e1), q2 = __fmaf_rn(-t, d[2], e2);
    return __fmaf_rn(q0, q0, __fmaf_rn(q1, q1, q2 * q2)) > thr2;
}
// the per-segment constants of far_from_capsule: 1 / |d|^2 and (rg + sqrt(3)/2 + 0.05)^2. A
// rounded t only moves the nearest point along the segment, which changes the distance by
// O(|d| * 2^-24)^2 -- far inside the 0.05-voxel margin.
__device__ __forceinline__ void far_consts(const float* w, float rg, float& iww, float& thr2) {
    const float ww = w[0] + w[1] + w[2];
    iww = ww > 0.0f ? 1.0f / ww : 0.0f;
    const float thr = rg + 0.91602540378f;
    thr2 = thr * thr;
}

// ---------------------------------------------------------------- emit

constexpr int EMIT_WARPS = 8;

// x / d for x < 2^24 (a segment has at most 2^24 candidates, §3) with m = floor((2^32-1)/d):
// umulhi(x, m) is floor(x/d) or one less (the error x (1 + d) / (d 2^32) < 2^-7), and the
// remainder test corrects it -- exact, without the integer-division sequence.
__device__ __forceinline__ uint32_t div_magic(uint32_t x, uint32_t d, uint32_t m) {
    uint32_t q = __umulhi(x, m);
    if (x - q * d >= d) q++;
    return q;
}
// Evaluates the first nq (<= 32) queued candidates, one per lane: the pinned predicate and
// l_r (§4), the exact S_acc contribution (segmented scan over lanes: queue order keeps the
// owner segments non-decreasing) and the binned append of in-grid, in-shard keys.
__device__ __forceinline__ void eval_queue(const int4* q, int nq, int lane, float (*sf)[32], const uint64_t* mtab,
                                           unsigned long long* sacc, uint64_t batch, const GridXf& g,
                                           const Shard& sh, const Bins& bins, uint64_t* __restrict__ keys,
                                           uint64_t* __restrict__ vals, unsigned* __restrict__ flags) {
    bool emit = false;
    uint64_t mkey = 0, val = 0;
    long long qv = 0;
    int o = 32;
    if (lane < nq) {
        const int4 e = q[lane];
        o = e.x;
        const int64_t i = e.y, j = e.z, k = e.w;
        Fib fo;
        for (int ax = 0; ax < 3; ax++) {
            fo.a[ax] = sf[ax][o];
            fo.w[ax] = sf[3 + ax][o];
            fo.iota[ax] = sf[6 + ax][o];
        }
        fo.r2 = sf[9][o];
        fo.moving = __float_as_uint(sf[10][o]);
        fo.len = sf[11][o];
        float ell;
        if (fiber_key(fo, i, j, k, ell)) {
            qv = q32(ell);
            if (i >= 0 && j >= 0 && k >= 0 && i < g.N && j < g.N && k < g.N) {
                mkey = morton3_tab(mtab, (uint32_t)i, (uint32_t)j, (uint32_t)k);
                const uint64_t cell = mkey >> sh.shift;
                if (cell >= sh.cell_lo && cell < sh.cell_hi) {
                    emit = true;
                    val = (batch * 32 + o) | ((uint64_t)__float_as_uint(ell) << 32);
                }
            }
        }
    }
#pragma unroll
    for (int dlt = 1; dlt < 32; dlt <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, qv, dlt);
        const int oy = __shfl_up_sync(0xffffffffu, o, dlt);
        if (lane >= dlt && oy == o) qv += y;
    }
    const int onext = __shfl_down_sync(0xffffffffu, o, 1);
    if (o < 32 && (lane == 31 || onext != o)) sacc[o] += (unsigned long long)qv;
    if (__ballot_sync(0xffffffffu, emit)) append_binned(emit, mkey, val, lane, bins, keys, vals, flags);
    __syncwarp();
}

// One warp per batch of 32 consecutive segments. The batch's candidate voxels (the
// unclamped AABB ranges, §3) are flattened and dealt round-robin to the 32 lanes, so every
// lane evaluates one (segment, voxel) candidate per step whatever the segment sizes.
// Keys add q(l_r) into the segment's exact S_acc (shared int64); in-grid, in-shard keys are
// compacted with a warp ballot and appended to the pair stream with one atomic per warp step.
__global__ void __launch_bounds__(EMIT_WARPS * 32, 4)
k_fiber_emit(const float* __restrict__ seg, const float* __restrict__ rad, uint64_t S, GridXf g, Shard sh,
             Bins bins, uint64_t* __restrict__ keys, uint64_t* __restrict__ vals, float4* __restrict__ ptab,
             unsigned* __restrict__ flags) {
    __shared__ float s_f[EMIT_WARPS][18][32];
    __shared__ int64_t s_u0[EMIT_WARPS][3][32];
    __shared__ uint32_t s_ex[EMIT_WARPS][4][32];   // x / y extents and their division magics
    __shared__ uint32_t s_start[EMIT_WARPS][32];
    __shared__ unsigned long long s_acc[EMIT_WARPS][32];
    __shared__ int4 s_q[EMIT_WARPS][64];   // survivor FIFO: (segment lane, i, j, k)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t nbatch = (S + 31) / 32;
    const float PI_F = 3.14159274101257324f;   // 0x40490FDB
    const bool whole = sh.cell_lo == 0 && sh.cell_hi == (1ull << (3 * g.logN - sh.shift));   // unsharded
    __shared__ uint64_t s_mtab[256];   // 8-bit Morton spreads
    mtab_init(s_mtab);
    const bool seg16 = (reinterpret_cast<uintptr_t>(seg) & 15u) == 0;
    for (uint64_t batch = blockIdx.x * (uint64_t)EMIT_WARPS + wib; batch < nbatch;
         batch += (uint64_t)gridDim.x * EMIT_WARPS) {
        const uint64_t p = batch * 32 + lane;
        uint32_t cnt = 0;
        Fib f;
        float d[3] = {0, 0, 0};
        float rg = 0.0f;
        // the batch's primitive tile (32 segments x 24 contiguous bytes) staged in the (empty)
        // survivor FIFO with 16-byte coalesced loads when the array is 16-byte aligned, then read
        // as 6 words per lane (measured neutral against 6 strided 4-byte loads per lane: the
        // kernel is issue-bound on the predicate)
        {
            float* st = reinterpret_cast<float*>(s_q[wib]);
            const uint64_t p0 = batch * 32;
            const int ns = S - p0 < 32 ? (int)(S - p0) : 32;
            if (seg16 && ns == 32) {
                const float4* src = reinterpret_cast<const float4*>(seg + 6 * p0);
                for (int w = lane; w < 48; w += 32) reinterpret_cast<float4*>(st)[w] = src[w];
            } else {
                for (int w = lane; w < 6 * ns; w += 32) st[w] = seg[6 * p0 + w];
            }
            __syncwarp();
        }
        if (p < S) {
            float s[6];
            for (int q = 0; q < 6; q++) s[q] = reinterpret_cast<const float*>(s_q[wib])[6 * lane + q];
            SegGeom G;
            seg_geom(g, s, rad[p], G);
            rg = G.rg;
            if (!G.culled && (whole || box_in_shard(G.e0, G.e1, sh))) {
                cnt = (uint32_t)((G.u1[0] - G.u0[0] + 1) * (G.u1[1] - G.u0[1] + 1) * (G.u1[2] - G.u0[2] + 1));
                for (int ax = 0; ax < 3; ax++) s_u0[wib][ax][lane] = G.u0[ax];
                s_ex[wib][0][lane] = (uint32_t)(G.u1[0] - G.u0[0] + 1);
                s_ex[wib][1][lane] = (uint32_t)(G.u1[1] - G.u0[1] + 1);
                s_ex[wib][2][lane] = 0xffffffffu / s_ex[wib][0][lane];
                s_ex[wib][3][lane] = 0xffffffffu / s_ex[wib][1][lane];
            }
            f.moving = 0;
            for (int ax = 0; ax < 3; ax++) {
                f.a[ax] = G.a[ax];
                d[ax] = G.b[ax] - G.a[ax];
                f.w[ax] = d[ax] * d[ax];
                if (f.w[ax] > 0.0f) { f.moving |= 1u << ax; f.iota[ax] = 1.0f / d[ax]; }
                else f.iota[ax] = 0.0f;
            }
            f.r2 = rg * rg;
            float ss = f.w[0] + f.w[1];
            ss = ss + f.w[2];
            f.len = sqrtf(ss);
            for (int ax = 0; ax < 3; ax++) {
                s_f[wib][ax][lane] = f.a[ax];
                s_f[wib][3 + ax][lane] = f.w[ax];
                s_f[wib][6 + ax][lane] = f.iota[ax];
            }
            s_f[wib][9][lane] = f.r2;
            s_f[wib][10][lane] = __uint_as_float(f.moving);
            s_f[wib][11][lane] = f.len;
            for (int ax = 0; ax < 3; ax++) s_f[wib][12 + ax][lane] = d[ax];
            s_f[wib][15][lane] = rg;
            far_consts(f.w, rg, s_f[wib][16][lane], s_f[wib][17][lane]);
        }
        __syncwarp();   // every lane has read its segment from the staging words
        // warp inclusive scan of the candidate counts
        uint32_t incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        s_start[wib][lane] = incl - cnt;
        s_acc[wib][lane] = 0ull;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        // Pass over the flattened candidates: cheap index math + conservative early reject;
        // survivors go to a per-warp FIFO in candidate order and are evaluated 32 at a time, so
        // the expensive pinned predicate runs on full warps.
        int qn = 0;
        for (uint32_t c0 = 0; c0 < total; c0 += 32) {
            const uint32_t c = c0 + lane;
            bool surv = false;
            int o = 0;
            int4 ent = make_int4(0, 0, 0, 0);
            if (c < total) {
#pragma unroll
                for (int step = 16; step; step >>= 1)
                    if (s_start[wib][o + step] <= c) o += step;
                const uint32_t local = c - s_start[wib][o];
                const uint32_t ex = s_ex[wib][0][o], ey = s_ex[wib][1][o];
                const uint32_t t = div_magic(local, ex, s_ex[wib][2][o]);
                const uint32_t tk = div_magic(t, ey, s_ex[wib][3][o]);
                const int64_t i = s_u0[wib][0][o] + (int64_t)(local - t * ex);
                const int64_t j = s_u0[wib][1][o] + (int64_t)(t - tk * ey);
                const int64_t k = s_u0[wib][2][o] + (int64_t)tk;
                float av[3], dv[3];
                for (int ax = 0; ax < 3; ax++) {
                    av[ax] = s_f[wib][ax][o];
                    dv[ax] = s_f[wib][12 + ax][o];
                }
                surv = !far_from_capsule(av, dv, s_f[wib][16][o], s_f[wib][17][o], i, j, k);
                ent = make_int4(o, (int)i, (int)j, (int)k);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, surv);
            if (surv) {
                VOX_DCHECK(qn + __popc(bal & ((1u << lane) - 1u)) < 64, 0);   // survivor FIFO
                s_q[wib][qn + __popc(bal & ((1u << lane) - 1u))] = ent;
            }
            qn += __popc(bal);
            __syncwarp();
            // the one evaluation site (the pinned predicate is inlined once): full rounds, and
            // after the last chunk the rest
            const bool last = c0 + 32 >= total;
            while (qn >= 32 || (last && qn > 0)) {
                const int m = qn < 32 ? qn : 32;
                eval_queue(s_q[wib], m, lane, s_f[wib], s_mtab, s_acc[wib], batch, g, sh, bins, keys, vals, flags);
                if (lane < qn - m) s_q[wib][lane] = s_q[wib][m + lane];
                qn -= m;
                __syncwarp();
            }
        }
        __syncwarp();
        if (p < S) {
            // §5 per-segment normalisation f_p = m_p / S_p and unit tangent
            const long long Sacc = (long long)s_acc[wib][lane];
            const float Sp = deq32(Sacc);
            float mp = PI_F * rg;
            mp = mp * rg;
            mp = mp * f.len;
            const float fp = Sacc > 0 ? mp / Sp : 0.0f;
            float4 e;
            e.x = f.len > 0.0f ? d[0] / f.len : 0.0f;
            e.y = f.len > 0.0f ? d[1] / f.len : 0.0f;
            e.z = f.len > 0.0f ? d[2] / f.len : 0.0f;
            e.w = fp;
            ptab[p] = e;
        }
        __syncwarp();
    }
}

cudaError_t launch_fiber_bound(vox_ctx* c, const float* seg, const float* rad, uint64_t S,
                               unsigned long long* cellW, int cell_log2) {
    const int threads = 256;
    uint64_t blocks = (S + threads - 1) / threads;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    k_fiber_bound<<<(unsigned)blocks, threads, 0, c->stream>>>(seg, rad, S, c->g, cell_log2, cellW, c->d_flags);
    c->st.launches++;
    return cudaGetLastError();
}

cudaError_t launch_fiber_emit(vox_ctx* c, const float* seg, const float* rad, uint64_t S, Shard sh, Bins bins,
                              uint64_t* keys, uint64_t* vals, float4* ptab) {
    const uint64_t nbatch = (S + 31) / 32;
    uint64_t blocks = (nbatch + EMIT_WARPS - 1) / EMIT_WARPS;
    if (blocks > (1ull << 30)) blocks = 1ull << 30;
    k_fiber_emit<<<(unsigned)blocks, EMIT_WARPS * 32, 0, c->stream>>>(seg, rad, S, c->g, sh, bins, keys, vals, ptab,
                                                                      c->d_flags);
    c->st.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- §13 sub-voxel density
__device__ __forceinline__ void fib_setup(Fib& f, float (&d)[3], const float* a, const float* b, float rg) {
    f.moving = 0;
    for (int ax = 0; ax < 3; ax++) {
        f.a[ax] = a[ax];
        d[ax] = b[ax] - a[ax];
        f.w[ax] = d[ax] * d[ax];
        if (f.w[ax] > 0.0f) { f.moving |= 1u << ax; f.iota[ax] = 1.0f / d[ax]; }
        else f.iota[ax] = 0.0f;
    }
    f.r2 = rg * rg;
    float ss = f.w[0] + f.w[1];
    ss = ss + f.w[2];
    f.len = sqrtf(ss);
}

// Warp per segment: its key voxels (the §4 predicate, as in emit), and for each key voxel the
// 512 sub-voxels, 16 per lane: the §4 predicate on the 8x grid, with conservative shortcuts
// (centre farther than R + sqrt(3)/2 + 0.1 fine voxels: no hit; the box within R - 0.1 of
// the segment point nearest its centre: hit) that the pinned fp32 decision cannot contradict (its deviation
// from the exact one is < 0.02 fine voxels at 8N <= 65536). The undecided sub-voxels of the
// segment's key voxels (about 16 per voxel) go to one per-warp ring and are evaluated 32 at a
// time across voxels, so the pinned predicate runs on full warps; up to DENS_PV key voxels are
// pending, each with its mask in shared memory, and their masks are OR-ed into the level-0
// masks when the pending set is full or the segment ends (a key absent from level 0 = another
// shard: skipped).
constexpr int DENS_PV = 32;          // pending key voxels per warp
constexpr int DENS_RING = 1024;     // undecided entries per warp (>= 31 + 512 live at once)

__global__ void __launch_bounds__(256, 2)
k_fiber_density(const float* __restrict__ seg, const float* __restrict__ rad, uint64_t S, GridXf g,
                const uint64_t* __restrict__ keys0, uint64_t n0, unsigned long long* __restrict__ masks) {
    __shared__ unsigned s_m[8][DENS_PV][16];   // per warp: the pending voxels' 512-bit masks
    __shared__ long long s_vidx[8][DENS_PV];   // their level-0 indices
    __shared__ int s_vc[8][DENS_PV][3];        // their voxel coordinates
    __shared__ uint16_t s_q[8][DENS_RING];     // per warp: undecided (slot << 9 | sub), a ring
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarp = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t p = warp; p < S; p += nwarp) {
        float s[6];
        for (int q = 0; q < 6; q++) s[q] = seg[6 * p + q];
        SegGeom G;
        seg_geom(g, s, rad[p], G);
        if (G.culled) continue;
        Fib f, f8;
        float d[3], d8[3], a8[3], b8[3];
        fib_setup(f, d, G.a, G.b, G.rg);
        for (int ax = 0; ax < 3; ax++) {
            a8[ax] = 8.0f * G.a[ax];
            b8[ax] = 8.0f * G.b[ax];
        }
        const float rg8 = 8.0f * G.rg;
        fib_setup(f8, d8, a8, b8, rg8);
        float iww, thr2, iww8, unused;
        far_consts(f.w, G.rg, iww, thr2);
        far_consts(f8.w, rg8, iww8, unused);
        // the centre is in the box: dist(segment, box) <= dist(segment, centre) and >= it - sqrt(3)/2
        const float far = rg8 + 0.96602540378f, near = rg8 - 0.1f;   // margins 0.1 fine voxel
        const float far2 = far * far, near2 = near > 0.0f ? near * near : -1.0f;
        const int64_t ex = G.e1[0] - G.e0[0] + 1, ey = G.e1[1] - G.e0[1] + 1, ez = G.e1[2] - G.e0[2] + 1;
        const int64_t ncand = ex * ey * ez;
        int pv = 0;                    // pending voxels
        unsigned head = 0, tail = 0;   // ring of undecided entries [head, tail)
        int64_t base = 0, i = 0, j = 0, k = 0;
        long long my_idx = -1;
        unsigned bal = 0;
        // one loop with a single evaluation site (the pinned predicate is inlined only once):
        // take the next key voxel of the segment, classify its sub-voxels, evaluate full rounds of
        // undecided ones; when the pending set is full or the segment is done, evaluate the rest
        // and OR the pending masks into level 0
        for (;;) {
            while (bal == 0 && base < ncand) {   // next chunk of candidates with key voxels
                const int64_t cidx = base + lane;
                bool key = false;
                if (cidx < ncand) {
                    i = G.e0[0] + cidx % ex;
                    j = G.e0[1] + (cidx / ex) % ey;
                    k = G.e0[2] + cidx / (ex * ey);
                    float ell;
                    key = !far_from_capsule(f.a, d, iww, thr2, i, j, k) && fiber_key(f, i, j, k, ell);
                }
                // every key lane searches its leaf at once (the searches' load latencies overlap)
                my_idx = key ? find_key(keys0, n0, morton3((uint32_t)i, (uint32_t)j, (uint32_t)k)) : -1;
                bal = __ballot_sync(0xffffffffu, my_idx >= 0);
                base += 32;
            }
            const bool done = bal == 0;
            if (!done) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1;
                const int64_t vi = __shfl_sync(0xffffffffu, i, src), vj = __shfl_sync(0xffffffffu, j, src),
                              vk = __shfl_sync(0xffffffffu, k, src);
                const long long idx = __shfl_sync(0xffffffffu, my_idx, src);
                const int slot = pv++;
                if (lane == 0) {
                    s_vidx[wib][slot] = idx;
                    s_vc[wib][slot][0] = (int)vi;
                    s_vc[wib][slot][1] = (int)vj;
                    s_vc[wib][slot][2] = (int)vk;
                }
                // classify the 512 sub-voxels (16 per lane): sure hits straight into the mask,
                // undecided ones queued
                // c2 = squared distance of the sub-voxel centre to the segment, box2 = squared
                // distance of the segment point nearest that centre to the sub-voxel box: the
                // segment-box distance lies in [sqrt(c2) - sqrt(3)/2, sqrt(box2)].
                // Centre offsets from the segment start: exact lattice offsets added to a per-voxel
                // base (the shortcut is conservative geometry, so its rounding need not match the
                // pinned predicate's; its error is far inside the 0.1 margin)
                const float e0 = (((float)(8 * vi) + 0.5f) - f8.a[0]) + (float)(lane & 7);
                const float e1a = (((float)(8 * vj) + 0.5f) - f8.a[1]) + (float)(lane >> 3);
                const float e1b = e1a + 4.0f;
                const float e2b = ((float)(8 * vk) + 0.5f) - f8.a[2];
                // (this classifier is conservative geometry, not the pinned predicate: fused
                // multiply-adds are fine here, their rounding is far inside the 0.1 margin)
                const float pa = __fmaf_rn(e1a, d8[1], e0 * d8[0]), pb = __fmaf_rn(e1b, d8[1], e0 * d8[0]);
                const unsigned lt = (1u << lane) - 1u;
                const unsigned tag = ((unsigned)slot << 9) | (unsigned)lane;   // sub-voxel lane + 32 q
                // rows q = 2 qz + h: z offset qz, y offset (lane >> 3) + 4 h (the two y values unrolled)
#pragma unroll 1
                for (int qz = 0; qz < 8; qz++) {
                    const float e2 = e2b + (float)qz;
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int q = 2 * qz + h;
                        const float e1 = h ? e1b : e1a;
                        float t = __fmaf_rn(e2, d8[2], h ? pb : pa) * iww8;
                        t = fminf(fmaxf(t, 0.0f), 1.0f);
                        const float q0 = __fmaf_rn(-t, d8[0], e0), q1 = __fmaf_rn(-t, d8[1], e1),
                                    q2 = __fmaf_rn(-t, d8[2], e2);
                        const float o0 = fmaxf(fabsf(q0) - 0.5f, 0.0f), o1 = fmaxf(fabsf(q1) - 0.5f, 0.0f),
                                    o2 = fmaxf(fabsf(q2) - 0.5f, 0.0f);
                        const float box2 = __fmaf_rn(o0, o0, __fmaf_rn(o1, o1, o2 * o2));
                        const float c2 = __fmaf_rn(q0, q0, __fmaf_rn(q1, q1, q2 * q2));
                        const bool sure = box2 < near2, open = !sure && !(c2 > far2);
                        const unsigned bs = __ballot_sync(0xffffffffu, sure);
                        const unsigned bo = __ballot_sync(0xffffffffu, open);
                        if (lane == 0) s_m[wib][slot][q] = bs;
                        if (open)
                            s_q[wib][(tail + __popc(bo & lt)) & (DENS_RING - 1)] = (uint16_t)(tag + 32u * q);
                        tail += __popc(bo);
                    }
                }
                __syncwarp();
            }
            const bool full = done || pv == DENS_PV;
            while (tail - head >= 32u || (full && head != tail)) {   // the one evaluation site
                const unsigned cnt = tail - head < 32u ? tail - head : 32u;
                if ((unsigned)lane < cnt) {
                    const unsigned e = s_q[wib][(head + lane) & (DENS_RING - 1)];
                    const int slot = e >> 9, sub = e & 511;
                    float ell;
                    if (fiber_key(f8, 8 * (int64_t)s_vc[wib][slot][0] + (sub & 7),
                                  8 * (int64_t)s_vc[wib][slot][1] + ((sub >> 3) & 7),
                                  8 * (int64_t)s_vc[wib][slot][2] + (sub >> 6), ell))
                        atomicOr(&s_m[wib][slot][sub >> 5], 1u << (sub & 31));
                }
                head += cnt;
                __syncwarp();
            }
            if (full) {
                for (int w = lane; w < pv * 8; w += 32) {
                    const int slot = w >> 3, q = w & 7;
                    const unsigned long long word = (unsigned long long)s_m[wib][slot][2 * q] |
                                                    ((unsigned long long)s_m[wib][slot][2 * q + 1] << 32);
                    if (word) atomicOr(&masks[8 * s_vidx[wib][slot] + q], word);
                }
                pv = 0;
                __syncwarp();
            }
            if (done) break;
        }
    }
}

cudaError_t launch_fiber_density(vox_ctx* c, const float* seg, const float* rad, uint64_t S) {
    const unsigned grid = (unsigned)std::min<uint64_t>((S + 7) / 8, 148ull * 16);
    k_fiber_density<<<grid ? grid : 1, 256, 0, c->stream>>>(seg, rad, S, c->g, c->lv[0].key, c->lv[0].n,
                                                          c->dmask[0]);
    c->st.launches++;
    return cudaGetLastError();
}

}  // namespace vox
