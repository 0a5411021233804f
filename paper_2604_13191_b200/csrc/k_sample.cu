// k_sample.cu -- the paper's sampling front end (docs/PREDICATES.md §12; SURVEY §8(f) NEXT-4;
// P:218-232 §3.2, §3.3): Catmull-Rom spline pieces sampled at t_s = (s + 1/2)/n
// ("equally distributed samples based in kernel indices") and triangles sampled with
// Heitz's low-distortion square -> triangle map, sample counts in proportion to the area of
// the largest triangle. Each sample is a (Morton key, contribution) pair appended to
// its Morton bin exactly like the exact-overlap pairs, so the binned reduce, the pyramid and
// SGGX-H are shared.
//
// Two passes per primitive kind: a bound pass counts the samples per bin (run-length
// aggregated per thread: consecutive samples of a primitive mostly share a bin), then the
// emit pass recomputes the samples and appends them (warp-matched atomics per bin).
#include "vox_internal.cuh"

namespace vox {

// ---------------------------------------------------------------- shared pieces
__device__ __forceinline__ bool sample_key(const GridXf& g, const float p[3], uint64_t& key) {
    uint32_t v[3];
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        const float f = floorf(p[ax]);
        if (!(f >= 0.0f) || !(f < g.Nf)) return false;   // outside [0, N): dropped
        v[ax] = (uint32_t)f;
    }
    key = morton3(v[0], v[1], v[2]);
    return true;
}

// per-thread run-length aggregation of bin counts
struct BinRun {
    unsigned long long bin = ~0ull, cnt = 0;
    __device__ __forceinline__ void add(unsigned long long b, unsigned long long* __restrict__ cellW) {
        if (b != bin) {
            if (cnt) atomicAdd(&cellW[bin], cnt);
            bin = b;
            cnt = 0;
        }
        cnt++;
    }
    __device__ __forceinline__ void flush(unsigned long long* __restrict__ cellW) {
        if (cnt) atomicAdd(&cellW[bin], cnt);
        cnt = 0;
    }
};

// ---------------------------------------------------------------- spline pieces (§12)
struct Piece {
    float G[4][3];
    float f;   // per-sample mass m_p / n
};

// controls -> grid (§1), m_p / n; false (with a flag) on bad input
__device__ __forceinline__ bool load_piece(const GridXf& g, const float* __restrict__ ctrl,
                                           const float* __restrict__ rad, uint64_t p, int n, Piece& P,
                                           unsigned* __restrict__ flags) {
    const float PI_F = 3.14159274101257324f;
    float c[12];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < 12; q++) {
        c[q] = ctrl[12 * p + q];
        bad |= !isfinite(c[q]);
    }
    const float r = rad[p];
    bad |= !isfinite(r);
    if (bad) {
        atomicOr(flags, VOX_EFLAG_NONFINITE);
        return false;
    }
    if (r < 0.0f) {
        atomicOr(flags, VOX_EFLAG_NEG_RADIUS);
        return false;
    }
#pragma unroll
    for (int m = 0; m < 4; m++)
#pragma unroll
        for (int ax = 0; ax < 3; ax++) P.G[m][ax] = to_grid(g, ax, c[3 * m + ax]);
    const float rg = to_grid_len(g, r);
    const float d0 = P.G[2][0] - P.G[1][0], d1 = P.G[2][1] - P.G[1][1], d2 = P.G[2][2] - P.G[1][2];
    float dd = d0 * d0 + d1 * d1;
    dd = dd + d2 * d2;
    float mp = PI_F * rg;
    mp = mp * rg;
    mp = mp * sqrtf(dd);
    P.f = mp / (float)n;
    return true;
}

__device__ __forceinline__ void spline_eval(const Piece& P, float t, float pos[3], float tan_[3]) {
    float dv[3];
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        const float c0 = 2.0f * P.G[1][ax];
        const float c1 = P.G[2][ax] - P.G[0][ax];
        const float c2 = ((2.0f * P.G[0][ax] - 5.0f * P.G[1][ax]) + 4.0f * P.G[2][ax]) - P.G[3][ax];
        const float c3 = ((3.0f * P.G[1][ax] - P.G[0][ax]) - 3.0f * P.G[2][ax]) + P.G[3][ax];
        pos[ax] = 0.5f * (((c3 * t + c2) * t + c1) * t + c0);
        dv[ax] = 0.5f * ((3.0f * c3 * t + 2.0f * c2) * t + c1);
    }
    float nn = dv[0] * dv[0] + dv[1] * dv[1];
    nn = nn + dv[2] * dv[2];
    const float nrm = sqrtf(nn);
#pragma unroll
    for (int ax = 0; ax < 3; ax++) tan_[ax] = nrm > 0.0f ? dv[ax] / nrm : 0.0f;
}

__global__ void k_spline_bound(const float* __restrict__ ctrl, const float* __restrict__ rad, uint64_t S, int n,
                               GridXf g, int bin_shift, unsigned long long* __restrict__ cellW,
                               unsigned* __restrict__ flags) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < S; p += (uint64_t)gridDim.x * blockDim.x) {
        Piece P;
        if (!load_piece(g, ctrl, rad, p, n, P, flags)) continue;
        BinRun run;
        for (int s = 0; s < n; s++) {
            const float t = ((float)s + 0.5f) / (float)n;
            float pos[3], tn[3];
            spline_eval(P, t, pos, tn);
            uint64_t key;
            if (sample_key(g, pos, key)) run.add(key >> bin_shift, cellW);
        }
        run.flush(cellW);
    }
}

__global__ void k_spline_emit(const float* __restrict__ ctrl, const float* __restrict__ rad, uint64_t S, int n,
                              GridXf g, Shard sh, Bins bins, uint64_t* __restrict__ keys,
                              uint64_t* __restrict__ vals, float4* __restrict__ ptab, unsigned* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarp = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t one = (uint64_t)__float_as_uint(1.0f) << 32;
    for (uint64_t p0 = warp * 32; p0 < S; p0 += nwarp * 32) {   // warp-uniform trip count
        const uint64_t p = p0 + lane;
        Piece P;
        const bool ok = p < S && load_piece(g, ctrl, rad, p, n, P, flags);
        for (int s = 0; s < n; s++) {
            bool emit = false;
            uint64_t key = 0;
            const uint64_t id = p * (uint64_t)n + s;   // < 2^32 (checked on the host)
            if (ok) {
                const float t = ((float)s + 0.5f) / (float)n;
                float pos[3], tn[3];
                spline_eval(P, t, pos, tn);
                if (sample_key(g, pos, key)) {
                    const uint64_t cell = key >> sh.shift;
                    emit = cell >= sh.cell_lo && cell < sh.cell_hi;
                    if (emit) ptab[id] = make_float4(tn[0], tn[1], tn[2], P.f);
                }
            }
            append_binned(emit, key, id | one, lane, bins, keys, vals, flags);
        }
    }
}

// ---------------------------------------------------------------- triangles (§12)
__device__ __forceinline__ void cross3s(const float* f, const float* g, float* out) {
    out[0] = f[1] * g[2] - f[2] * g[1];
    out[1] = f[2] * g[0] - f[0] * g[2];
    out[2] = f[0] * g[1] - f[1] * g[0];
}

struct TriS {
    float g[9];
    float A;
    float dh[3];
};

// grid vertices, whole area (§7 area formula, one fan term), direction (§7); false on bad input
__device__ __forceinline__ bool load_tri(const GridXf& gx, const float* __restrict__ tri,
                                         const float* __restrict__ dirs, uint64_t t, TriS& T,
                                         unsigned* __restrict__ flags) {
    bool bad = false;
    float v[9];
#pragma unroll
    for (int q = 0; q < 9; q++) {
        v[q] = tri[9 * t + q];
        bad |= !isfinite(v[q]);
    }
    float w[3];
    if (dirs) {
#pragma unroll
        for (int q = 0; q < 3; q++) {
            w[q] = dirs[3 * t + q];
            bad |= !isfinite(w[q]);
        }
    }
    if (bad) {
        atomicOr(flags, VOX_EFLAG_NONFINITE);
        return false;
    }
#pragma unroll
    for (int q = 0; q < 9; q++) T.g[q] = to_grid(gx, q % 3, v[q]);
    if (!dirs) {
        float f1[3], f2[3];
#pragma unroll
        for (int ax = 0; ax < 3; ax++) {
            f1[ax] = T.g[3 + ax] - T.g[ax];
            f2[ax] = T.g[6 + ax] - T.g[3 + ax];
        }
        cross3s(f1, f2, w);
    }
    float nn = w[0] * w[0] + w[1] * w[1];
    nn = nn + w[2] * w[2];
    const float nrm = sqrtf(nn);
    if (dirs && !(nrm > 0.0f)) {
        atomicOr(flags, VOX_EFLAG_ZERO_DIR);
        return false;
    }
#pragma unroll
    for (int ax = 0; ax < 3; ax++) T.dh[ax] = nrm > 0.0f ? w[ax] / nrm : 0.0f;
    float e1[3], e2[3], cr[3];
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        e1[ax] = T.g[3 + ax] - T.g[ax];
        e2[ax] = T.g[6 + ax] - T.g[ax];
    }
    cross3s(e1, e2, cr);
    const float a0 = 0.0f + cr[0], a1 = 0.0f + cr[1], a2 = 0.0f + cr[2];
    float aa = a0 * a0 + a1 * a1;
    aa = aa + a2 * a2;
    T.A = 0.5f * sqrtf(aa);
    return true;
}

__device__ __forceinline__ int tri_nsamp(float A, float Amax, int budget) {
    if (!(A > 0.0f)) return 0;
    const int k = (int)floorf((A / Amax) * (float)budget + 0.5f);
    return k < 1 ? 1 : k;
}

__device__ __forceinline__ void tri_point(const TriS& T, int s, int nt, float p[3]) {
    const float u0 = ((float)s + 0.5f) / (float)nt;
    const float x = (float)s * 0.618034f;
    const float u1 = x - floorf(x);
    float b0, b1;
    if (u1 > u0) {   // Heitz 2019 low-distortion map (both branches are a few selects)
        b0 = 0.5f * u0;
        b1 = u1 - b0;
    } else {
        b1 = 0.5f * u1;
        b0 = u0 - b1;
    }
    const float b2 = (1.0f - b0) - b1;
#pragma unroll
    for (int ax = 0; ax < 3; ax++) p[ax] = (b0 * T.g[ax] + b1 * T.g[3 + ax]) + b2 * T.g[6 + ax];
}

__global__ void k_tri_amax(const float* __restrict__ tri, const float* __restrict__ dirs, uint64_t T, GridXf gx,
                           unsigned* __restrict__ amax_bits, unsigned* __restrict__ flags) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        TriS S;
        if (!load_tri(gx, tri, dirs, t, S, flags)) continue;
        atomicMax(amax_bits, __float_as_uint(S.A));   // A >= 0: bit order = value order
    }
}

__global__ void k_tris_bound(const float* __restrict__ tri, const float* __restrict__ dirs, uint64_t T, int budget,
                             GridXf gx, const unsigned* __restrict__ amax_bits, int bin_shift,
                             unsigned long long* __restrict__ cellW, unsigned* __restrict__ flags) {
    const float Amax = __uint_as_float(*amax_bits);
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        TriS S;
        if (!load_tri(gx, tri, dirs, t, S, flags)) continue;
        const int nt = tri_nsamp(S.A, Amax, budget);
        BinRun run;
        for (int s = 0; s < nt; s++) {
            float p[3];
            tri_point(S, s, nt, p);
            uint64_t key;
            if (sample_key(gx, p, key)) run.add(key >> bin_shift, cellW);
        }
        run.flush(cellW);
    }
}

__global__ void k_tris_emit(const float* __restrict__ tri, const float* __restrict__ dirs, uint64_t T, int budget,
                            GridXf gx, const unsigned* __restrict__ amax_bits, Shard sh, Bins bins,
                            uint64_t* __restrict__ keys, uint64_t* __restrict__ vals, float4* __restrict__ ptab,
                            unsigned* __restrict__ flags) {
    const float Amax = __uint_as_float(*amax_bits);
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarp = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t one = (uint64_t)__float_as_uint(1.0f) << 32;
    for (uint64_t t0 = warp * 32; t0 < T; t0 += nwarp * 32) {
        const uint64_t t = t0 + lane;
        TriS S;
        int nt = 0;
        if (t < T && load_tri(gx, tri, dirs, t, S, flags)) {
            nt = tri_nsamp(S.A, Amax, budget);
            if (nt > 0) ptab[t] = make_float4(S.dh[0], S.dh[1], S.dh[2], S.A / (float)nt);
        }
        const int nmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)nt);
        for (int s = 0; s < nmax; s++) {
            bool emit = false;
            uint64_t key = 0;
            if (s < nt) {
                float p[3];
                tri_point(S, s, nt, p);
                if (sample_key(gx, p, key)) {
                    const uint64_t cell = key >> sh.shift;
                    emit = cell >= sh.cell_lo && cell < sh.cell_hi;
                }
            }
            append_binned(emit, key, t | one, lane, bins, keys, vals, flags);
        }
    }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_spline_bound(vox_ctx* c, const float* ctrl, const float* rad, uint64_t S, int n,
                                unsigned long long* cellW, int bin_log2) {
    const unsigned grid = (unsigned)std::min<uint64_t>((S + 255) / 256, 148ull * 16);
    k_spline_bound<<<grid ? grid : 1, 256, 0, c->stream>>>(ctrl, rad, S, n, c->g, 3 * bin_log2, cellW, c->d_flags);
    c->st.launches++;
    return cudaGetLastError();
}

cudaError_t launch_spline_emit(vox_ctx* c, const float* ctrl, const float* rad, uint64_t S, int n, Shard sh,
                               Bins bins, uint64_t* keys, uint64_t* vals, float4* ptab) {
    const unsigned grid = (unsigned)std::min<uint64_t>((S + 255) / 256, 148ull * 16);
    k_spline_emit<<<grid ? grid : 1, 256, 0, c->stream>>>(ctrl, rad, S, n, c->g, sh, bins, keys, vals, ptab,
                                                        c->d_flags);
    c->st.launches++;
    return cudaGetLastError();
}

cudaError_t launch_tris_bound(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, int budget,
                              unsigned* amax_bits, unsigned long long* cellW, int bin_log2) {
    const unsigned grid = (unsigned)std::min<uint64_t>((T + 255) / 256, 148ull * 16);
    cudaError_t e = cudaMemsetAsync(amax_bits, 0, 4, c->stream);
    if (e != cudaSuccess) return e;
    k_tri_amax<<<grid ? grid : 1, 256, 0, c->stream>>>(tri, dirs, T, c->g, amax_bits, c->d_flags);
    k_tris_bound<<<grid ? grid : 1, 256, 0, c->stream>>>(tri, dirs, T, budget, c->g, amax_bits, 3 * bin_log2, cellW,
                                                       c->d_flags);
    c->st.launches += 2;
    return cudaGetLastError();
}

cudaError_t launch_tris_emit(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, int budget,
                             const unsigned* amax_bits, Shard sh, Bins bins, uint64_t* keys, uint64_t* vals,
                             float4* ptab) {
    const unsigned grid = (unsigned)std::min<uint64_t>((T + 255) / 256, 148ull * 16);
    k_tris_emit<<<grid ? grid : 1, 256, 0, c->stream>>>(tri, dirs, T, budget, c->g, amax_bits, sh, bins, keys, vals,
                                                       ptab, c->d_flags);
    c->st.launches++;
    return cudaGetLastError();
}

}  // namespace vox
