// k_tri.cu -- triangles: cull/bin (k_tri_bound) and separating-axis triangle-box test +
// half-open clipped area emit (k_tri_emit). docs/PREDICATES.md §1, §3, §6, §7 (north star:
// triangle-box SAT; P:225-228 area-weighted triangle sampling whose continuous limit is the
// clipped area; P:179 face normals, P:183/P:549 tangent mode).

#include "vox_internal.cuh"

namespace vox {

struct TriGeom {
    float g[9];
    bool culled;
    int64_t e0[3], e1[3];
};

__device__ __forceinline__ void tri_geom(const GridXf& gx, const float* v, TriGeom& G) {
    for (int m = 0; m < 3; m++)
        for (int ax = 0; ax < 3; ax++) G.g[3 * m + ax] = to_grid(gx, ax, v[3 * m + ax]);
    G.culled = false;
    const float Nhi = gx.Nf + 1.0f;
    for (int ax = 0; ax < 3; ax++) {
        float lo = pmin(pmin(G.g[ax], G.g[3 + ax]), G.g[6 + ax]);
        float hi = pmax(pmax(G.g[ax], G.g[3 + ax]), G.g[6 + ax]);
        if (!(hi >= -1.0f) || !(lo <= Nhi)) { G.culled = true; return; }
        int64_t c0 = (int64_t)ceilf(lo) - 1, c1 = (int64_t)floorf(hi);
        G.e0[ax] = c0 < 0 ? 0 : c0;
        G.e1[ax] = c1 > gx.N - 1 ? gx.N - 1 : c1;
        if (G.e0[ax] > G.e1[ax]) G.culled = true;
    }
}

__device__ __forceinline__ void cross3(const float* f, const float* g, float* o) {
    o[0] = f[1] * g[2] - f[2] * g[1];
    o[1] = f[2] * g[0] - f[0] * g[2];
    o[2] = f[0] * g[1] - f[1] * g[0];
}

// §7 direction: face normal of the grid-space triangle or the caller's dir; returns nrm.
__device__ __forceinline__ float tri_dir(const float* g, const float* dir, float* dh) {
    float w[3];
    if (dir) {
        w[0] = dir[0]; w[1] = dir[1]; w[2] = dir[2];
    } else {
        float f1[3], f2[3];
        for (int ax = 0; ax < 3; ax++) { f1[ax] = g[3 + ax] - g[ax]; f2[ax] = g[6 + ax] - g[3 + ax]; }
        cross3(f1, f2, w);
    }
    float nn = w[0] * w[0] + w[1] * w[1];
    nn = nn + w[2] * w[2];
    const float nrm = sqrtf(nn);
    for (int ax = 0; ax < 3; ax++) dh[ax] = nrm > 0.0f ? w[ax] / nrm : 0.0f;
    return nrm;
}

__global__ void k_tri_bound(const float* __restrict__ tri, const float* __restrict__ dirs, uint64_t T, GridXf gx,
                            int cell_shift, unsigned long long* __restrict__ cellW, unsigned* __restrict__ flags) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T;
         t += (uint64_t)gridDim.x * blockDim.x) {
        float v[9];
        bool bad = false;
        for (int q = 0; q < 9; q++) { v[q] = tri[9 * t + q]; bad |= !isfinite(v[q]); }
        if (dirs) {
            float d[3] = {dirs[3 * t], dirs[3 * t + 1], dirs[3 * t + 2]};
            for (int q = 0; q < 3; q++) bad |= !isfinite(d[q]);
            if (!bad) {
                float nn = d[0] * d[0] + d[1] * d[1];
                nn = nn + d[2] * d[2];
                if (!(sqrtf(nn) > 0.0f)) { atomicOr(flags, VOX_EFLAG_ZERO_DIR); continue; }
            }
        }
        if (bad) { atomicOr(flags, VOX_EFLAG_NONFINITE); continue; }
        TriGeom G;
        tri_geom(gx, v, G);
        if (G.culled) continue;
        const int s = cell_shift;
        for (int64_t cz = G.e0[2] >> s; cz <= G.e1[2] >> s; cz++) {
            int64_t nz = min(G.e1[2], ((cz + 1) << s) - 1) - max(G.e0[2], cz << s) + 1;
            for (int64_t cy = G.e0[1] >> s; cy <= G.e1[1] >> s; cy++) {
                int64_t ny = min(G.e1[1], ((cy + 1) << s) - 1) - max(G.e0[1], cy << s) + 1;
                for (int64_t cx = G.e0[0] >> s; cx <= G.e1[0] >> s; cx++) {
                    int64_t nx = min(G.e1[0], ((cx + 1) << s) - 1) - max(G.e0[0], cx << s) + 1;
                    atomicAdd(&cellW[morton3((uint32_t)cx, (uint32_t)cy, (uint32_t)cz)],
                              (unsigned long long)(nx * ny * nz));
                }
            }
        }
    }
}

// ---------------------------------------------------------------- §6 SAT (closed box)

__device__ __forceinline__ bool sep3(float p0, float p1, float p2, float rad) {
    const float mn = pmin(pmin(p0, p1), p2);
    const float mx = pmax(pmax(p0, p1), p2);
    return mn > rad || mx < -rad;
}

__device__ __forceinline__ bool tri_box_sat(const float* g, int64_t i, int64_t j, int64_t k) {
    const float h = 0.5f;
    const float c[3] = {(float)i + 0.5f, (float)j + 0.5f, (float)k + 0.5f};
    float v[3][3], e[3][3];
#pragma unroll
    for (int m = 0; m < 3; m++)
#pragma unroll
        for (int ax = 0; ax < 3; ax++) v[m][ax] = g[3 * m + ax] - c[ax];
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        e[0][ax] = v[1][ax] - v[0][ax];
        e[1][ax] = v[2][ax] - v[1][ax];
        e[2][ax] = v[0][ax] - v[2][ax];
    }
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const float ex = e[q][0], ey = e[q][1], ez = e[q][2];
        const float fx = fabsf(ex), fy = fabsf(ey), fz = fabsf(ez);
        float p[3];
        for (int m = 0; m < 3; m++) p[m] = ez * v[m][1] - ey * v[m][2];
        if (sep3(p[0], p[1], p[2], fz * h + fy * h)) return false;
        for (int m = 0; m < 3; m++) p[m] = ex * v[m][2] - ez * v[m][0];
        if (sep3(p[0], p[1], p[2], fz * h + fx * h)) return false;
        for (int m = 0; m < 3; m++) p[m] = ey * v[m][0] - ex * v[m][1];
        if (sep3(p[0], p[1], p[2], fy * h + fx * h)) return false;
    }
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        const float mn = pmin(pmin(v[0][ax], v[1][ax]), v[2][ax]);
        const float mx = pmax(pmax(v[0][ax], v[1][ax]), v[2][ax]);
        if (mn > h || mx < -h) return false;
    }
    float n[3], vmin[3], vmax[3];
    cross3(e[0], e[1], n);
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        if (n[ax] > 0.0f) { vmin[ax] = -h - v[0][ax]; vmax[ax] = h - v[0][ax]; }
        else { vmin[ax] = h - v[0][ax]; vmax[ax] = -h - v[0][ax]; }
    }
    float dmin = n[0] * vmin[0] + n[1] * vmin[1];
    dmin = dmin + n[2] * vmin[2];
    if (dmin > 0.0f) return false;
    float dmax = n[0] * vmax[0] + n[1] * vmax[1];
    dmax = dmax + n[2] * vmax[2];
    return !(dmax < 0.0f);
}

// ---------------------------------------------------------------- §7 clipped area (half-open box)

constexpr int MAXPOLY = 12;

__device__ __forceinline__ int clip_one(const float (*in)[3], int n, float (*out)[3], int ax, float c, bool upper) {
    int o = 0;
    for (int m = 0; m < n; m++) {
        const float* cur = in[m];
        const float* prev = in[m == 0 ? n - 1 : m - 1];
        const bool cin = upper ? (cur[ax] < c) : (cur[ax] >= c);
        const bool pin = upper ? (prev[ax] < c) : (prev[ax] >= c);
        if (cin != pin) {
            const float s = (c - prev[ax]) / (cur[ax] - prev[ax]);
            for (int b = 0; b < 3; b++) out[o][b] = (b == ax) ? c : prev[b] + s * (cur[b] - prev[b]);
            o++;
        }
        if (cin) {
            out[o][0] = cur[0]; out[o][1] = cur[1]; out[o][2] = cur[2];
            o++;
        }
    }
    return o;
}

__device__ float tri_clip_area(const float* g, int64_t i, int64_t j, int64_t k) {
    float P[MAXPOLY][3], Q[MAXPOLY][3];
    for (int m = 0; m < 3; m++)
        for (int ax = 0; ax < 3; ax++) P[m][ax] = g[3 * m + ax];
    int n = 3;
    const float lo[3] = {(float)i, (float)j, (float)k};
    const float hi[3] = {(float)(i + 1), (float)(j + 1), (float)(k + 1)};
    for (int ax = 0; ax < 3; ax++) {
        n = clip_one(P, n, Q, ax, lo[ax], false);
        if (n < 3) return 0.0f;
        n = clip_one(Q, n, P, ax, hi[ax], true);
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

// ---------------------------------------------------------------- emit

// Per-triangle setup (grid-space vertices, clamped candidate box, prim table entry) and the
// candidate count; an exclusive scan of the counts then lets the emit kernel deal fixed-size
// chunks of the global candidate space to warps, so one huge triangle or a handful of
// triangles still spread over the whole GPU.
struct TriSetup {
    float g[9];
    int e0[3];
    unsigned ex, ey;
    unsigned pad;
};

__global__ void k_tri_setup(const float* __restrict__ tri, const float* __restrict__ dirs, uint64_t T, GridXf gx,
                            Shard sh, TriSetup* __restrict__ ts, unsigned long long* __restrict__ tcnt,
                            float4* __restrict__ ptab) {
    const bool whole = sh.cell_lo == 0 && sh.cell_hi == (1ull << (3 * gx.logN - sh.shift));   // unsharded
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        float v[9];
        for (int q = 0; q < 9; q++) v[q] = tri[9 * t + q];
        TriGeom G;
        tri_geom(gx, v, G);
        float dh[3];
        tri_dir(G.g, dirs ? dirs + 3 * t : nullptr, dh);
        ptab[t] = make_float4(dh[0], dh[1], dh[2], 1.0f);
        TriSetup s;
        for (int q = 0; q < 9; q++) s.g[q] = G.g[q];
        unsigned long long cnt = 0;
        if (!G.culled && (whole || box_in_shard(G.e0, G.e1, sh))) {   // no key in this shard: skipped
            for (int ax = 0; ax < 3; ax++) s.e0[ax] = (int)G.e0[ax];
            s.ex = (unsigned)(G.e1[0] - G.e0[0] + 1);
            s.ey = (unsigned)(G.e1[1] - G.e0[1] + 1);
            cnt = (unsigned long long)s.ex * s.ey * (unsigned long long)(G.e1[2] - G.e0[2] + 1);
        } else {
            s.e0[0] = s.e0[1] = s.e0[2] = 0;
            s.ex = s.ey = 1;
        }
        s.pad = 0;
        ts[t] = s;
        tcnt[t] = cnt;
    }
}

constexpr int TRI_WARPS = 4;
constexpr int TRI_CHUNK = 256;   // candidates per warp work item

__device__ __forceinline__ uint64_t tri_upper(const unsigned long long* __restrict__ toff, uint64_t lo, uint64_t hi,
                                              unsigned long long c) {
    // last t in [lo, hi) with toff[t] <= c
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (toff[mid] <= c) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Warps take TRI_CHUNK consecutive candidates of the global (triangle-major) candidate space;
// each lane locates its triangle by a binary search bounded by the chunk's first/last triangle.
// Keys (SAT, §6) in the shard go to a per-warp FIFO in candidate order; the clipped area (§7)
// is evaluated 32 queued keys at a time (full warps: about a quarter of the candidates are
// keys, so evaluating them in place left three lanes in four idle), then the (key, prim |
// area) pairs are appended to their bins.
__device__ __forceinline__ void tri_eval_queue(const int4* q, int nq, int lane, const TriSetup* __restrict__ ts,
                                               const Bins& bins, uint64_t* __restrict__ keys,
                                               uint64_t* __restrict__ vals, unsigned* __restrict__ flags) {
    bool emit = false;
    uint64_t mkey = 0, val = 0;
    if (lane < nq) {
        const int4 e = q[lane];
        const uint32_t t = (uint32_t)e.x;   // prim indices are 32-bit (the pair value packs them so)
        float g[9];
#pragma unroll
        for (int x = 0; x < 9; x++) g[x] = ts[t].g[x];
        const float A = tri_clip_area(g, e.y, e.z, e.w);
        mkey = morton3((uint32_t)e.y, (uint32_t)e.z, (uint32_t)e.w);
        val = (uint64_t)t | ((uint64_t)__float_as_uint(A) << 32);
        emit = true;
    }
    if (__ballot_sync(0xffffffffu, emit)) append_binned(emit, mkey, val, lane, bins, keys, vals, flags);
    __syncwarp();
}

__global__ void __launch_bounds__(TRI_WARPS * 32)
k_tri_emit(const TriSetup* __restrict__ ts, const unsigned long long* __restrict__ toff, uint64_t T, GridXf gx,
           Shard sh, Bins bins, uint64_t* __restrict__ keys, uint64_t* __restrict__ vals,
           unsigned* __restrict__ flags) {
    __shared__ int4 s_q[TRI_WARPS][64];   // key FIFO: (triangle, i, j, k)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const unsigned long long total = toff[T];
    const unsigned long long nchunk = (total + TRI_CHUNK - 1) / TRI_CHUNK;
    for (unsigned long long ch = blockIdx.x * (unsigned long long)TRI_WARPS + wib; ch < nchunk;
         ch += (unsigned long long)gridDim.x * TRI_WARPS) {
        const unsigned long long cb = ch * TRI_CHUNK;
        const unsigned long long ce = cb + TRI_CHUNK < total ? cb + TRI_CHUNK : total;
        uint64_t tlo = 0, thi = 0;
        if (lane == 0) {
            tlo = tri_upper(toff, 0, T, cb);
            thi = tri_upper(toff, tlo, T, ce - 1) + 1;
        }
        tlo = __shfl_sync(0xffffffffu, tlo, 0);
        thi = __shfl_sync(0xffffffffu, thi, 0);
        int qn = 0;
        for (unsigned long long c0 = cb; c0 < ce; c0 += 32) {
            const unsigned long long c = c0 + lane;
            bool key = false;
            int4 ent = make_int4(0, 0, 0, 0);
            if (c < ce) {
                const uint64_t t = tri_upper(toff, tlo, thi, c);
                const TriSetup s = ts[t];
                const unsigned long long local = c - toff[t];
                const unsigned long long q = local / s.ex;
                const int64_t i = s.e0[0] + (int64_t)(local - q * s.ex);
                const int64_t j = s.e0[1] + (int64_t)(q % s.ey);
                const int64_t k = s.e0[2] + (int64_t)(q / s.ey);
                if (tri_box_sat(s.g, i, j, k)) {
                    const uint64_t cell = morton3((uint32_t)i, (uint32_t)j, (uint32_t)k) >> sh.shift;
                    key = cell >= sh.cell_lo && cell < sh.cell_hi;
                    ent = make_int4((int)t, (int)i, (int)j, (int)k);
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, key);
            if (key) s_q[wib][qn + __popc(bal & ((1u << lane) - 1u))] = ent;   // qn < 32 here: < 64
            qn += __popc(bal);
            __syncwarp();
            // the one evaluation site of the clipped area: full rounds, after the last chunk the rest
            const bool last = c0 + 32 >= ce;
            while (qn >= 32 || (last && qn > 0)) {
                const int m = qn < 32 ? qn : 32;
                tri_eval_queue(s_q[wib], m, lane, ts, bins, keys, vals, flags);
                if (lane < qn - m) s_q[wib][lane] = s_q[wib][m + lane];
                qn -= m;
                __syncwarp();
            }
        }
    }
}

cudaError_t launch_tri_bound(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, unsigned long long* cellW,
                             int cell_log2) {
    const int threads = 256;
    uint64_t blocks = (T + threads - 1) / threads;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    k_tri_bound<<<(unsigned)blocks, threads, 0, c->stream>>>(tri, dirs, T, c->g, cell_log2, cellW, c->d_flags);
    c->st.launches++;
    return cudaGetLastError();
}

cudaError_t launch_tri_emit(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, Shard sh, Bins bins,
                            uint64_t* keys, uint64_t* vals, float4* ptab) {
    TriSetup* ts = nullptr;
    unsigned long long *tcnt = nullptr, *toff = nullptr;
    cudaError_t e;
    if ((e = dalloc(c, (void**)&ts, T * sizeof(TriSetup))) != cudaSuccess) return e;
    if ((e = dalloc(c, (void**)&tcnt, (T + 1) * 8)) != cudaSuccess) return e;
    if ((e = dalloc(c, (void**)&toff, (T + 1) * 8)) != cudaSuccess) return e;
    uint64_t blocks = (T + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    k_tri_setup<<<(unsigned)blocks, 256, 0, c->stream>>>(tri, dirs, T, c->g, sh, ts, tcnt, ptab);
    if ((e = cudaMemsetAsync(tcnt + T, 0, 8, c->stream)) != cudaSuccess) return e;
    if ((e = scan_excl_u64(c, tcnt, toff, T + 1)) != cudaSuccess) return e;
    k_tri_emit<<<148u * 16, TRI_WARPS * 32, 0, c->stream>>>(ts, toff, T, c->g, sh, bins, keys, vals, c->d_flags);
    c->st.launches += 2;   // + the scan's own
    e = cudaGetLastError();
    dfree(c, toff);
    dfree(c, tcnt);
    dfree(c, ts);
    return e;
}

// ---------------------------------------------------------------- §13 sub-voxel density
// Warp per triangle: key voxels by the §6 SAT, then per key voxel the 512 sub-voxels (16 per
// lane) by the §6 SAT on the 8x grid, skipping (no hit) sub-voxels whose centre is farther
// than sqrt(3)/2 + 0.25 fine voxels from the triangle's plane (GPU-only shortcut; the pinned
// SAT cannot report overlap there).
__global__ void __launch_bounds__(256, 2)
k_tri_density(const float* __restrict__ tri, uint64_t T, GridXf gx, const uint64_t* __restrict__ keys0,
              uint64_t n0, unsigned long long* __restrict__ masks) {
    __shared__ unsigned s_m[8][16];        // per warp: the voxel's 512-bit mask
    __shared__ uint16_t s_q[8][512];       // per warp: sub-voxels to test
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarp = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = warp; t < T; t += nwarp) {
        float v[9];
        for (int q = 0; q < 9; q++) v[q] = tri[9 * t + q];
        TriGeom G;
        tri_geom(gx, v, G);
        if (G.culled) continue;
        float g8[9];
        for (int q = 0; q < 9; q++) g8[q] = 8.0f * G.g[q];
        // plane of the fine triangle (shortcut geometry only)
        float e1[3], e2[3], n[3];
        for (int ax = 0; ax < 3; ax++) {
            e1[ax] = g8[3 + ax] - g8[ax];
            e2[ax] = g8[6 + ax] - g8[ax];
        }
        cross3(e1, e2, n);
        const float nn = sqrtf(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        const float lim = 1.11602540378f * nn;   // (sqrt(3)/2 + 0.25) |n|
        const int64_t ex = G.e1[0] - G.e0[0] + 1, ey = G.e1[1] - G.e0[1] + 1, ez = G.e1[2] - G.e0[2] + 1;
        const int64_t ncand = ex * ey * ez;
        for (int64_t base = 0; base < ncand; base += 32) {
            const int64_t cidx = base + lane;
            int64_t i = 0, j = 0, k = 0;
            bool key = false;
            if (cidx < ncand) {
                i = G.e0[0] + cidx % ex;
                j = G.e0[1] + (cidx / ex) % ey;
                k = G.e0[2] + cidx / (ex * ey);
                key = tri_box_sat(G.g, i, j, k);
            }
            // every key lane searches its leaf at once (the searches' load latencies overlap)
            const long long my_idx = key ? find_key(keys0, n0, morton3((uint32_t)i, (uint32_t)j, (uint32_t)k)) : -1;
            unsigned bal = __ballot_sync(0xffffffffu, my_idx >= 0);
            while (bal) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1;
                const int64_t vi = __shfl_sync(0xffffffffu, i, src), vj = __shfl_sync(0xffffffffu, j, src),
                              vk = __shfl_sync(0xffffffffu, k, src);
                const long long idx = __shfl_sync(0xffffffffu, my_idx, src);
                // sub-voxels off the plane's slab are no hit; the others are queued and tested
                // by the pinned SAT 32 at a time
                int nq = 0;
                if (lane < 16) s_m[wib][lane] = 0u;
#pragma unroll 1
                for (int q = 0; q < 16; q++) {
                    const int sub = lane + 32 * q;
                    const int64_t x = 8 * vi + (sub & 7), y = 8 * vj + ((sub >> 3) & 7), z = 8 * vk + (sub >> 6);
                    const float pd = (((float)x + 0.5f) - g8[0]) * n[0] + (((float)y + 0.5f) - g8[1]) * n[1] +
                                     (((float)z + 0.5f) - g8[2]) * n[2];
                    const bool open = !(nn > 0.0f && fabsf(pd) > lim);
                    const unsigned bo = __ballot_sync(0xffffffffu, open);
                    if (open) s_q[wib][nq + __popc(bo & ((1u << lane) - 1u))] = (uint16_t)sub;
                    nq += __popc(bo);
                }
                __syncwarp();
#pragma unroll 1
                for (int b0 = 0; b0 < nq; b0 += 32) {
                    if (b0 + lane < nq) {
                        const int sub = s_q[wib][b0 + lane];
                        if (tri_box_sat(g8, 8 * vi + (sub & 7), 8 * vj + ((sub >> 3) & 7), 8 * vk + (sub >> 6)))
                            atomicOr(&s_m[wib][sub >> 5], 1u << (sub & 31));
                    }
                }
                __syncwarp();
                if (lane < 8) {
                    const unsigned long long word =
                        (unsigned long long)s_m[wib][2 * lane] | ((unsigned long long)s_m[wib][2 * lane + 1] << 32);
                    if (word) atomicOr(&masks[8 * idx + lane], word);
                }
                __syncwarp();
            }
        }
    }
}

cudaError_t launch_tri_density(vox_ctx* c, const float* tri, uint64_t T) {
    const unsigned grid = (unsigned)std::min<uint64_t>((T + 7) / 8, 148ull * 16);
    k_tri_density<<<grid ? grid : 1, 256, 0, c->stream>>>(tri, T, c->g, c->lv[0].key, c->lv[0].n, c->dmask[0]);
    c->st.launches++;
    return cudaGetLastError();
}

}  // namespace vox
