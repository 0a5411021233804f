// k_reduce.cu -- gathering (§3.3 "ordered by second level block ID ... detect the
// vector positions where the ID changes") as a device radix sort of (Morton key, payload)
// pairs followed by a segmented reduction into exact fixed-point accumulators
// (docs/PREDICATES.md §8). Also merges a new leaf set into an existing one (D19).
//
// Round-1 scaffold: the sort and the two scans use CUB (header-only, CUDA 12.9); the
// per-voxel accumulation is ours. To be replaced by a fused bucket-sort + reduce kernel.
#include <cub/cub.cuh>

#include "vox_internal.cuh"

namespace vox {

__global__ void k_heads(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ flags) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// heads -> start offsets of each run; start[V] = n.
__global__ void k_starts(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ incl, uint64_t n,
                         uint32_t* __restrict__ start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (flags[i]) start[incl[i] - 1] = (uint32_t)i;
        if (i == n - 1) start[incl[i]] = (uint32_t)n;
    }
}

// One thread per voxel: exact sum of q(contribution) over its run of pairs (§5, §7, §8).
__global__ void k_accum(const uint32_t* __restrict__ start, uint64_t V, const uint64_t* __restrict__ keys,
                        const uint64_t* __restrict__ vals, const float4* __restrict__ ptab,
                        uint64_t* __restrict__ okey, long long* __restrict__ oacc) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = start[v], e = start[v + 1];
        long long a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0;
        for (uint32_t i = s; i < e; i++) {
            const uint64_t val = vals[i];
            const float4 pt = ptab[(uint32_t)val];
            const float w = __uint_as_float((uint32_t)(val >> 32));
            const float mass = pt.w * w;
            const float mx = mass * pt.x, my = mass * pt.y, mz = mass * pt.z;
            a0 += q32(mass);
            a1 += q32(mx * pt.x);
            a2 += q32(my * pt.y);
            a3 += q32(mz * pt.z);
            a4 += q32(mx * pt.y);
            a5 += q32(mx * pt.z);
            a6 += q32(my * pt.z);
        }
        okey[v] = keys[s];
        long long* o = oacc + 7 * v;
        o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3; o[4] = a4; o[5] = a5; o[6] = a6;
    }
}

// One thread per voxel of a merge: sum the accumulator rows of its run (rows < n0 come from
// the old leaf, the rest from the new one).
__global__ void k_sum_rows(const uint32_t* __restrict__ start, uint64_t V, const uint64_t* __restrict__ keys,
                           const uint32_t* __restrict__ idx, const long long* __restrict__ accA, uint64_t n0,
                           const long long* __restrict__ accB, uint64_t* __restrict__ okey,
                           long long* __restrict__ oacc) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = start[v], e = start[v + 1];
        long long a[7] = {0, 0, 0, 0, 0, 0, 0};
        for (uint32_t i = s; i < e; i++) {
            const uint64_t r = idx[i];
            const long long* src = r < n0 ? accA + 7 * r : accB + 7 * (r - n0);
            for (int q = 0; q < 7; q++) a[q] += src[q];
        }
        okey[v] = keys[s];
        for (int q = 0; q < 7; q++) oacc[7 * v + q] = a[q];
    }
}

__global__ void k_iota(uint32_t* __restrict__ p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

static unsigned grid_for(uint64_t n, int threads = 256) {
    uint64_t b = (n + threads - 1) / threads;
    if (b > 148ull * 32) b = 148ull * 32;
    if (b == 0) b = 1;
    return (unsigned)b;
}

#define CK(x)                                                      \
    do {                                                           \
        cudaError_t e_ = (x);                                      \
        if (e_ != cudaSuccess) {                                   \
            c->err = std::string(#x) + ": " + cudaGetErrorString(e_); \
            return e_ == cudaErrorMemoryAllocation ? VOX_ERR_OOM : VOX_ERR_CUDA; \
        }                                                          \
    } while (0)

// Runs of equal keys in sorted keys[0..n): returns V and start[V+1] (caller frees).
static vox_status find_runs(vox_ctx* c, const uint64_t* keys, uint64_t n, uint32_t** start_out, uint64_t* V_out) {
    uint32_t *flags = nullptr, *incl = nullptr, *start = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    CK(dalloc(c, (void**)&flags, n * 4));
    CK(dalloc(c, (void**)&incl, n * 4));
    k_heads<<<grid_for(n), 256, 0, c->stream>>>(keys, n, flags);
    c->st.launches++;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, flags, incl, (int64_t)n, c->stream));
    CK(dalloc(c, &tmp, tb));
    CK(cub::DeviceScan::InclusiveSum(tmp, tb, flags, incl, (int64_t)n, c->stream));
    c->st.launches += 2;   // scan init + scan
    uint32_t V32 = 0;
    CK(cudaMemcpyAsync(&V32, incl + n - 1, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(dalloc(c, (void**)&start, ((uint64_t)V32 + 1) * 4));
    k_starts<<<grid_for(n), 256, 0, c->stream>>>(flags, incl, n, start);
    c->st.launches++;
    dfree(c, tmp);
    dfree(c, incl);
    dfree(c, flags);
    *start_out = start;
    *V_out = V32;
    return VOX_OK;
}

static vox_status merge_into_leaf(vox_ctx* c, uint64_t* nkey, long long* nacc, uint64_t V) {
    Level& L0 = c->lv[0];
    if (L0.n == 0) {
        free_level(c, L0);
        L0.n = V;
        L0.key = nkey;
        L0.acc = nacc;
    } else {
        timer_begin(c, c->t_merge);
        const uint64_t n0 = L0.n, tot = n0 + V;
        uint64_t *k0 = nullptr, *k1 = nullptr;
        uint32_t *i0 = nullptr, *i1 = nullptr;
        void* tmp = nullptr;
        size_t tb = 0;
        CK(dalloc(c, (void**)&k0, tot * 8));
        CK(dalloc(c, (void**)&k1, tot * 8));
        CK(dalloc(c, (void**)&i0, tot * 4));
        CK(dalloc(c, (void**)&i1, tot * 4));
        CK(cudaMemcpyAsync(k0, L0.key, n0 * 8, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(k0 + n0, nkey, V * 8, cudaMemcpyDeviceToDevice, c->stream));
        k_iota<<<grid_for(tot), 256, 0, c->stream>>>(i0, tot);
        c->st.launches++;
        cub::DoubleBuffer<uint64_t> dk(k0, k1);
        cub::DoubleBuffer<uint32_t> dv(i0, i1);
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int64_t)tot, 0, 3 * c->g.logN, c->stream));
        CK(dalloc(c, &tmp, tb));
        CK(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int64_t)tot, 0, 3 * c->g.logN, c->stream));
        c->st.launches += 2 + (3 * c->g.logN + 7) / 8;
        uint32_t* start = nullptr;
        uint64_t VM = 0;
        vox_status s = find_runs(c, dk.Current(), tot, &start, &VM);
        if (s != VOX_OK) return s;
        uint64_t* mkey = nullptr;
        long long* macc = nullptr;
        CK(dalloc(c, (void**)&mkey, VM * 8));
        CK(dalloc(c, (void**)&macc, VM * 56));
        k_sum_rows<<<grid_for(VM), 256, 0, c->stream>>>(start, VM, dk.Current(), dv.Current(), L0.acc, n0, nacc,
                                                         mkey, macc);
        c->st.launches++;
        dfree(c, start);
        dfree(c, tmp);
        dfree(c, k0); dfree(c, k1); dfree(c, i0); dfree(c, i1);
        dfree(c, nkey);
        dfree(c, nacc);
        free_level(c, L0);
        L0.n = VM;
        L0.key = mkey;
        L0.acc = macc;
        timer_end(c, c->t_merge);
    }
    CK(dalloc(c, (void**)&L0.mass, (L0.n ? L0.n : 1) * 4));
    CK(dalloc(c, (void**)&L0.m6, (L0.n ? L0.n : 1) * 24));
    CK(launch_finalize(c, L0, false));
    return VOX_OK;
}

vox_status reduce_pairs(vox_ctx* c, uint64_t* keys, uint64_t* keys_alt, uint64_t* vals, uint64_t* vals_alt,
                        uint64_t P, const float4* ptab) {
    if (P == 0) return VOX_OK;
    timer_begin(c, c->t_sort);
    cub::DoubleBuffer<uint64_t> dk(keys, keys_alt), dv(vals, vals_alt);
    void* tmp = nullptr;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int64_t)P, 0, 3 * c->g.logN, c->stream));
    CK(dalloc(c, &tmp, tb));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int64_t)P, 0, 3 * c->g.logN, c->stream));
    c->st.launches += 2 + (3 * c->g.logN + 7) / 8;   // histogram + exclusive sum + one onesweep pass per 8 bits
    timer_end(c, c->t_sort);
    dfree(c, tmp);
    timer_begin(c, c->t_reduce);
    uint32_t* start = nullptr;
    uint64_t V = 0;
    vox_status s = find_runs(c, dk.Current(), P, &start, &V);
    if (s != VOX_OK) return s;
    uint64_t* nkey = nullptr;
    long long* nacc = nullptr;
    CK(dalloc(c, (void**)&nkey, V * 8));
    CK(dalloc(c, (void**)&nacc, V * 56));
    k_accum<<<grid_for(V), 256, 0, c->stream>>>(start, V, dk.Current(), dv.Current(), ptab, nkey, nacc);
    c->st.launches++;
    dfree(c, start);
    timer_end(c, c->t_reduce);
    c->st.voxels = V;
    return merge_into_leaf(c, nkey, nacc, V);
}

}  // namespace vox
