// k_lod.cu -- the 2x2x2 Morton pyramid with per-parent SGGX-H clustering
// (§4.4 Eq. similarity; docs/PREDICATES.md §9), fp32 finalisation of levels, and
// the fixed-size level records used by the multi-GPU gather.
//
// Parents are runs of equal key>>3 in the sorted child level (Morton order is hierarchical,
// so no re-sort). One warp per parent: lanes 0..6 sum the 7 accumulators exactly; the
// children's lobes are gathered into shared memory; if more than K remain, SGGX-H runs with
// lane = slice for sigma (32 slices = 32 lanes) and lane = pair for distances and argmin.
#include <cmath>

#include "vox_internal.cuh"

namespace vox {

VOX_DEBUG_TU(lod)

__constant__ float c_coef[VOX_SLICES][6];

// PREDICATES §9 slice table: spherical Fibonacci on the upper hemisphere, evaluated in fp64,
// rounded to fp32; Theta_k from the fp32 theta in fp64 (exact products), rounded to fp32.
void host_theta(float theta[32][3], float coef[32][6]) {
    const double pi = 3.14159265358979323846;
    const double golden_angle = pi * (3.0 - std::sqrt(5.0));
    for (int k = 0; k < 32; k++) {
        const double z = 1.0 - (k + 0.5) / 32.0;
        const double rho = std::sqrt(1.0 - z * z);
        const double phi = k * golden_angle;
        theta[k][0] = (float)(rho * std::cos(phi));
        theta[k][1] = (float)(rho * std::sin(phi));
        theta[k][2] = (float)z;
        const double x = theta[k][0], y = theta[k][1], zz = theta[k][2];
        coef[k][0] = (float)(x * x);
        coef[k][1] = (float)(y * y);
        coef[k][2] = (float)(zz * zz);
        coef[k][3] = (float)(2.0 * x * y);
        coef[k][4] = (float)(2.0 * x * zz);
        coef[k][5] = (float)(2.0 * y * zz);
    }
}

void upload_theta(vox_ctx* c) {
    float theta[32][3], coef[32][6];
    host_theta(theta, coef);
    cudaMemcpyToSymbolAsync(c_coef, coef, sizeof(coef), 0, cudaMemcpyHostToDevice, c->stream);
}

constexpr unsigned INF_BITS = 0x7f800000u;

// pair index t = j(j-1)/2 + i for i < j (pairs with j < n are the prefix t < n(n-1)/2)
__device__ __forceinline__ int pair_t(int i, int j) { return j * (j - 1) / 2 + i; }


// ---------------------------------------------------------------- per-level prep
// One thread per parent: exact naive aggregate, fp32 copies, the number n of
// dendrogram leaves (children's lobes with w != 0, D17). Parents with n <= K are final here
// (their lobes are copied in child-slot order); the others are counted per n so that the
// SGGX-H kernels get them grouped by n (uniform work per warp).
template <int K>
__global__ void k_lod_prep(const long long* __restrict__ cacc,
                           const uint8_t* __restrict__ cncl, const long long* __restrict__ cclacc, int leaf,
                           const uint32_t* __restrict__ start, uint64_t V, long long* __restrict__ pacc,
                           uint8_t* __restrict__ pncl, long long* __restrict__ pclacc,
                           uint8_t* __restrict__ nlob, unsigned* __restrict__ hist) {
    constexpr int MAXN = 8 * K;
    __shared__ unsigned s_hist[MAXN + 1];
    for (int x = threadIdx.x; x <= MAXN; x += blockDim.x) s_hist[x] = 0;
    __syncthreads();
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < V; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c0 = start[p], c1 = start[p + 1];
        long long sum[7] = {0, 0, 0, 0, 0, 0, 0};
        int n = 0;
        for (uint32_t x = c0; x < c1; x++) {
#pragma unroll
            for (int e = 0; e < 7; e++) sum[e] += cacc[7 * (uint64_t)x + e];
            // stored lobes always have w > 0 (leaf lobes need mass > 0, merges add positives),
            // so the dendrogram leaves are counted without reading them; should a w = 0 lobe
            // ever appear, the copy below and the SGGX-H gathers still drop it (only the bucket
            // choice would differ, not the result)
            if (leaf) n += cacc[7 * (uint64_t)x] > 0;
            else n += cncl[x];
        }
#pragma unroll
        for (int e = 0; e < 7; e++) pacc[7 * p + e] = sum[e];
        nlob[p] = (uint8_t)n;
        if (n <= K) {
            int slot = 0;
            for (uint32_t x = c0; x < c1; x++) {
                if (leaf) {
                    if (cacc[7 * (uint64_t)x] > 0) {
                        for (int e = 0; e < 7; e++) pclacc[(p * K + slot) * 7 + e] = cacc[7 * (uint64_t)x + e];
                        slot++;
                    }
                } else {
                    for (int q = 0; q < cncl[x]; q++) {
                        const long long* src = cclacc + ((uint64_t)x * K + q) * 7;
                        if (src[0] == 0) continue;
                        for (int e = 0; e < 7; e++) pclacc[(p * K + slot) * 7 + e] = src[e];
                        slot++;
                    }
                }
            }
            // unused slots are written as zeros: they are never read, but skipping them leaves
            // partial sectors that cost more than the bytes (measured)
            for (int q = slot; q < K; q++)
                for (int e = 0; e < 7; e++) pclacc[(p * K + q) * 7 + e] = 0;
            pncl[p] = (uint8_t)slot;
        } else {
            atomicAdd(&s_hist[n], 1u);
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x <= MAXN; x += blockDim.x)
        if (s_hist[x]) atomicAdd(&hist[x], s_hist[x]);
}

// Level-1 prep (children are leaves): one warp per PREP_PAR consecutive parents. Their
// children are one contiguous block of leaf rows; lane 0 fetches it into shared memory with a
// single bulk async copy (cp.async.bulk, completion on an mbarrier), double-buffered so the
// next block's copy is in flight while this one is reduced. Each lane then reduces its own
// parent from shared memory, and the outputs are staged and written back as contiguous words.
// Same arithmetic as k_lod_prep (exact integer sums). The copy is 16-byte aligned by starting
// up to one 8-byte word early and rounding the size up; every device buffer carries >= 64 B of
// allocation slack (dalloc), so the rounded tail stays inside the allocation.
#ifndef PREP_WARPS_N
#define PREP_WARPS_N 4
#endif
#ifndef PREP_PAR_N
#define PREP_PAR_N 16
#endif
constexpr int PREP_WARPS = PREP_WARPS_N;
constexpr int PREP_PAR = PREP_PAR_N;                  // parents per warp-iteration
constexpr int PREP_ROWW = 8 * PREP_PAR * 7 + 2;       // staged words per buffer (+ alignment)
constexpr int PREP_WARP_WORDS = 2 * PREP_ROWW + PREP_PAR * 7 + 2;   // + acc staging; lobes added per K

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(b), "r"(phase)
            : "memory");
    }
}

template <int K>
__global__ void __launch_bounds__(PREP_WARPS * 32)
k_lod_prep_leaf(const long long* __restrict__ cacc,
                const uint32_t* __restrict__ start, uint64_t V, long long* __restrict__ pacc,
                uint8_t* __restrict__ pncl, long long* __restrict__ pclacc,
                uint8_t* __restrict__ nlob, unsigned* __restrict__ hist) {
    constexpr int MAXN = 8 * K;
    extern __shared__ __align__(16) long long s_dyn[];   // per warp: 2 x rows | acc | lobes
    __shared__ unsigned s_hist[MAXN + 1];
    __shared__ uint64_t s_bar[PREP_WARPS][2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int x = threadIdx.x; x <= MAXN; x += blockDim.x) s_hist[x] = 0;
    if (lane == 0) {
        mbar_init(&s_bar[wib][0], 1);
        mbar_init(&s_bar[wib][1], 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    long long* wbase = s_dyn + (size_t)wib * (PREP_WARP_WORDS + PREP_PAR * K * 7);
    long long* sacc = wbase + 2 * PREP_ROWW;
    long long* slob = sacc + PREP_PAR * 7 + 2;
    const uint64_t stride = (uint64_t)gridDim.x * PREP_WARPS * PREP_PAR;
    uint64_t p0 = (blockIdx.x * (uint64_t)PREP_WARPS + wib) * PREP_PAR;
    // issue the bulk copy of block q0's children into buffer b; returns the word offset
    // issue the bulk copy of the block whose child range [s0, s1) is given into buffer b
    auto issue = [&](uint64_t s0, uint64_t s1, int b) {
        const uint64_t w0 = 7 * s0, w1 = 7 * s1;
        const uint64_t a0 = w0 & ~1ull;                      // 16-byte aligned start word
        const unsigned bytes = (unsigned)(((w1 - a0) * 8 + 15) & ~15ull);
        if (bytes) {
            mbar_arrive_tx(&s_bar[wib][b], bytes);
            bulk_g2s(wbase + (size_t)b * PREP_ROWW, cacc + a0, bytes, &s_bar[wib][b]);
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&s_bar[wib][b])) : "memory");
        }
    };
    // child ranges of a block: start[q0], start[min(q0 + PREP_PAR, V)] (lane 0 only)
    auto range = [&](uint64_t q0, uint64_t& s0, uint64_t& s1) {
        s0 = start[q0];
        s1 = start[q0 + PREP_PAR < V ? q0 + PREP_PAR : V];
    };
    uint64_t ns0 = 0, ns1 = 0;   // the range of the block after the next (prefetched a step ahead)
    if (lane == 0 && p0 < V) {
        uint64_t s0, s1;
        range(p0, s0, s1);
        issue(s0, s1, 0);
        if (p0 + stride < V) range(p0 + stride, ns0, ns1);
    }
    unsigned phase = 0;   // bit b: parity of buffer b's next completion
    for (int it = 0; p0 < V; p0 += stride, it++) {
        const int b = it & 1;
        if (lane == 0 && p0 + stride < V) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(ns0, ns1, b ^ 1);
            if (p0 + 2 * stride < V) range(p0 + 2 * stride, ns0, ns1);   // consumed next iteration
        }
        const uint64_t pe = p0 + PREP_PAR < V ? p0 + PREP_PAR : V;
        const int np = (int)(pe - p0);
        const uint32_t cs = start[p0];
        int c0 = 0, c1 = 0;
        if (lane < np) {
            c0 = (int)(start[p0 + lane] - cs);
            c1 = (int)(start[p0 + lane + 1] - cs);
        }
        mbar_wait(&s_bar[wib][b], (phase >> b) & 1u);
        phase ^= 1u << b;
        const long long* rows = wbase + (size_t)b * PREP_ROWW + ((7 * (uint64_t)cs) & 1);
        VOX_DCHECK(lane >= np || 7 * c1 + (int)((7 * (uint64_t)cs) & 1) <= PREP_ROWW, 7);   // staged child rows
        bool hard = false;
        if (lane < np) {
            const uint64_t p = p0 + lane;
            long long sum[7] = {0, 0, 0, 0, 0, 0, 0};
            int n = 0;
            for (int x = c0; x < c1; x++) {
#pragma unroll
                for (int e = 0; e < 7; e++) sum[e] += rows[7 * x + e];
                n += rows[7 * x] > 0;
            }
#pragma unroll
            for (int e = 0; e < 7; e++) sacc[7 * lane + e] = sum[e];
            nlob[p] = (uint8_t)n;
            hard = n > K;
            int slot = 0;
            for (int x = c0; x < c1 && slot < K; x++) {
                if (rows[7 * x] > 0) {
#pragma unroll
                    for (int e = 0; e < 7; e++) slob[(lane * K + slot) * 7 + e] = rows[7 * x + e];
                    slot++;
                }
            }
            for (int q = slot; q < K; q++)
#pragma unroll
                for (int e = 0; e < 7; e++) slob[(lane * K + q) * 7 + e] = 0;
            if (!hard) pncl[p] = (uint8_t)slot;
            else atomicAdd(&s_hist[n], 1u);
        }
        const unsigned hmask = __ballot_sync(0xffffffffu, hard);
        __syncwarp();
        // coalesced write-back: accumulators, lobes of the final (n <= K) parents (zero slots
        // included: whole sectors)
        for (int w = lane; w < np * 7; w += 32) pacc[7 * p0 + w] = sacc[w];
        for (int w = lane; w < np * K * 7; w += 32) {
            if ((hmask >> (w / (K * 7))) & 1u) continue;
            pclacc[(uint64_t)p0 * K * 7 + w] = slob[w];
        }
        __syncwarp();
    }
    __syncthreads();
    for (int x = threadIdx.x; x <= MAXN; x += blockDim.x)
        if (s_hist[x]) atomicAdd(&hist[x], s_hist[x]);
}

// Exclusive offsets of the per-n buckets (ascending n) and the split between the quad
// kernel (n <= 8) and the warp kernel (n > 8). counts = {n_small, n_total}.
// Also accumulates the level's algorithmic SGGX-H work into work[3] (sigma evaluations:
// n + (n - K); distance evaluations: n(n-1)/2 + sum over merges of (m - 2); hard parents).
__global__ void k_bucket_init(const unsigned* __restrict__ hist, int K, int maxn, unsigned* __restrict__ cursor,
                              unsigned* __restrict__ counts, unsigned long long* __restrict__ work) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    unsigned off = 0, small = 0, mid = 0;
    unsigned long long sg = 0, dd = 0, hp = 0;
    for (int n = K + 1; n <= maxn; n++) {
        cursor[n] = off;
        off += hist[n];
        if (n <= 8) small = off;
        if (n <= 16) mid = off;
        // evaluations actually needed: n initial sigmas and pairs, then a new sigma and a new
        // row for every merge but the last (after it, nothing reads sigma or D)
        unsigned long long d = (unsigned long long)n * (n - 1) / 2;
        for (int m = n; m > K + 1; m--) d += (unsigned long long)(m - 2);
        sg += (unsigned long long)hist[n] * (unsigned long long)(2 * n - K - 1);
        dd += (unsigned long long)hist[n] * d;
        hp += hist[n];
    }
    counts[0] = small;   // [0, small): n <= 8 (group kernel)
    counts[1] = mid;     // [small, mid): 9 <= n <= 16 (half-warp kernel)
    counts[2] = off;     // [mid, off): n > 16 (warp kernel)
    if (work) {
        work[0] += sg;
        work[1] += dd;
        work[2] += hp;
    }
}

constexpr int SCATTER_PER_THREAD = 8;

// Hard parents (n > K) into their bucket; block-local counting keeps global atomics per bin.
__global__ void k_bucket_scatter(const uint8_t* __restrict__ nlob, uint64_t V, int K, int maxn,
                                 unsigned* __restrict__ cursor, uint32_t* __restrict__ list) {
    __shared__ unsigned s_cnt[65], s_base[65];
    for (int x = threadIdx.x; x <= maxn; x += blockDim.x) s_cnt[x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * blockDim.x * SCATTER_PER_THREAD;
    uint8_t nn[SCATTER_PER_THREAD];
#pragma unroll
    for (int r = 0; r < SCATTER_PER_THREAD; r++) {
        const uint64_t p = base + (uint64_t)r * blockDim.x + threadIdx.x;
        nn[r] = p < V ? nlob[p] : 0;
        if (nn[r] > K) atomicAdd(&s_cnt[nn[r]], 1u);
    }
    __syncthreads();
    for (int x = threadIdx.x; x <= maxn; x += blockDim.x) {
        s_base[x] = s_cnt[x] ? atomicAdd(&cursor[x], s_cnt[x]) : 0;
        s_cnt[x] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < SCATTER_PER_THREAD; r++) {
        if (nn[r] > K) {
            const uint64_t p = base + (uint64_t)r * blockDim.x + threadIdx.x;
            list[s_base[nn[r]] + atomicAdd(&s_cnt[nn[r]], 1u)] = (uint32_t)p;
        }
    }
}

// Dendrogram leaves of parent p (levels >= 2): children's stored lobes in child-slot order,
// w = 0 dropped (D17). One lane per (child, lobe slot) -- 8 children x K slots <= 32 lanes
// for K <= 4, looped otherwise -- compacted by ballot so the order is exactly the serial one.
template <int K>
__device__ __forceinline__ int gather_lobes(const uint32_t* __restrict__ start, const uint8_t* __restrict__ cncl,
                                            const long long* __restrict__ cclacc, uint64_t p, int lane,
                                            unsigned mask, long long* out) {
    const uint32_t c0 = start[p], c1 = start[p + 1];
    const int slots = (int)(c1 - c0) * K;
    int n = 0;
    for (int b = 0; b < 8 * K; b += 32) {
        const int sl = b + lane;
        bool has = false;
        const long long* src = nullptr;
        if (sl < slots) {
            const uint64_t x = c0 + sl / K;
            const int q = sl % K;
            src = cclacc + (x * K + q) * 7;
            has = q < cncl[x] && src[0] != 0;
        }
        const unsigned bal = __ballot_sync(mask, has);
        if (has) {
            const int c = n + __popc(bal & ((1u << lane) - 1u));
            VOX_DCHECK(c < 8 * K, 3);
#pragma unroll
            for (int e = 0; e < 7; e++) out[7 * c + e] = src[e];
        }
        n += __popc(bal);
    }
    return n;
}

// ---------------------------------------------------------------- SGGX-H, n <= 8 ("quad")
// Four parents per warp, eight lanes per parent. Lane l of a group owns slices l, l+8,
// l+16, l+24 of every lobe's sigma (a float4 per lobe in shared memory). A distance is formed as the pinned tree
// pairs it -- s[l] = d[l] + d[l+16], s[l+8] = d[l+8] + d[l+24], s[l] = s[l] + s[l+8] in
// registers, then the last three tree levels by xor-shuffles inside the group -- and kept in
// a shared 28-entry table per parent; the lexicographic argmin (d, i, j) is a group reduce.
constexpr int QUAD_WARPS = 4;
#ifndef QUAD_MINB
#define QUAD_MINB 7
#endif

__device__ __forceinline__ float part4(const float* a, const float* b) {
    return (fabsf(a[0] - b[0]) + fabsf(a[2] - b[2])) + (fabsf(a[1] - b[1]) + fabsf(a[3] - b[3]));
}
// Eight distances at once: slot s of lane l holds the lane's part4 of pair (s ^ l); at step h
// a lane keeps the slots with bit h clear and adds the partner's slot s | h, which holds the
// same pair (s ^ l = (s | h) ^ (l ^ h)). Lane l ends with pair l's sum, and each addition is
// the pinned tree's s[x] + s[x + h] (fp32 addition is commutative): bit-identical to the
// per-pair xor reduce, with 7 shuffles per 8 pairs instead of 24 and no selects.
__device__ __forceinline__ float group_sum8x8(float (&v)[8]) {
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
        for (int s = 0; s < h; s++) v[s] = v[s] + __shfl_xor_sync(0xffffffffu, v[s + h], h);
    return v[0];
}

template <int K>
__global__ void __launch_bounds__(QUAD_WARPS * 32, QUAD_MINB)
k_sggxh_quad(const uint32_t* __restrict__ list, const unsigned* __restrict__ counts,
             const long long* __restrict__ cacc, const uint8_t* __restrict__ cncl,
             const long long* __restrict__ cclacc, int leaf, const uint32_t* __restrict__ start,
             uint8_t* __restrict__ pncl, long long* __restrict__ pclacc) {
    __shared__ long long s_lobe[QUAD_WARPS][4][8][7];
    __shared__ __align__(16) float s_S[QUAD_WARPS][4][8][6];
    __shared__ float s_D[QUAD_WARPS][4][28];
    __shared__ __align__(16) float4 s_sg[QUAD_WARPS][4][8][8];   // [group][lobe][lane]: the lane's 4 slices
    __shared__ uint16_t s_pair[32];   // 28 pairs; entries 28..31 pad the last batch of 8
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int l = lane & 7, g = lane >> 3;
    if (threadIdx.x < 32) {
        int j = 1;
        while ((j + 1) * j / 2 <= (int)threadIdx.x) j++;
        s_pair[threadIdx.x] = threadIdx.x < 28 ? (uint16_t)((((int)threadIdx.x - j * (j - 1) / 2) << 8) | j) : (uint16_t)1;
    }
    __syncthreads();
    long long(*lobe)[7] = s_lobe[wib][g];
    float(*Sg)[6] = s_S[wib][g];
    float* D = s_D[wib][g];
    __shared__ __align__(16) float s_cfl[8][4][6];   // [l][q][e] = coefficient e of slice l + 8 q
    for (int x = threadIdx.x; x < 8 * 4 * 6; x += blockDim.x) {
        const int ll = x / 24, q = (x / 6) % 4, e = x % 6;
        s_cfl[ll][q][e] = c_coef[ll + 8 * q][e];
    }
    __syncthreads();
    // coefficients of this lane's slices l, l+8, l+16, l+24, read from shared memory at each use
    // (keeps 24 registers free: occupancy is what the serial merge chains need)
    const float2(*cf)[3] = reinterpret_cast<const float2(*)[3]>(s_cfl[l]);
    const unsigned small = counts[0];
    const unsigned nquad = (small + 3) / 4;
    for (unsigned qd = blockIdx.x * QUAD_WARPS + wib; qd < nquad; qd += gridDim.x * QUAD_WARPS) {
        const unsigned idx = 4 * qd + g;
        const bool valid = idx < small;
        const uint32_t p = valid ? list[idx] : 0;
        int n = 0;
        if (leaf) {
            uint32_t c0 = 0;
            int nch = 0;
            if (valid) {
                c0 = start[p];
                nch = (int)(start[p + 1] - c0);
            }
            long long a[7] = {0, 0, 0, 0, 0, 0, 0};
            if (l < nch) {
#pragma unroll
                for (int e = 0; e < 7; e++) a[e] = cacc[7 * (uint64_t)(c0 + l) + e];
            }
            const bool has = l < nch && a[0] > 0;
            const unsigned gm = (__ballot_sync(0xffffffffu, has) >> (8 * g)) & 0xffu;
            n = __popc(gm);
            if (has) {
                const int c = __popc(gm & ((1u << l) - 1u));
#pragma unroll
                for (int e = 0; e < 7; e++) lobe[c][e] = a[e];
            }
        } else {
            // 8 lanes x (child, lobe slot) rounds; n <= 8 here
            n = 0;
            uint32_t c0 = 0, c1 = 0;
            if (valid) {
                c0 = start[p];
                c1 = start[p + 1];
            }
            const int slots = (int)(c1 - c0) * K;
            for (int b = 0; b < 8 * K; b += 8) {
                const int sl = b + l;
                bool has = false;
                const long long* src = nullptr;
                if (sl < slots) {
                    const uint64_t x = c0 + sl / K;
                    const int q = sl % K;
                    src = cclacc + (x * K + q) * 7;
                    has = q < cncl[x] && src[0] != 0;
                }
                const unsigned gm = (__ballot_sync(0xffffffffu, has) >> (8 * g)) & 0xffu;
                if (has) {
                    const int c = n + __popc(gm & ((1u << l) - 1u));
                    VOX_DCHECK(c < 8, 4);
#pragma unroll
                    for (int e = 0; e < 7; e++) lobe[c][e] = src[e];
                }
                n += __popc(gm);
            }
        }
        __syncwarp();
        const int nmax = __reduce_max_sync(0xffffffffu, valid ? n : 0);
        if (valid && l < n) {
            const float wf = deq32(lobe[l][0]);
#pragma unroll
            for (int e = 0; e < 6; e++) Sg[l][e] = deq32(lobe[l][1 + e]) / wf;
        }
        __syncwarp();
        // the lane's 4 sigma slices of every lobe live in shared memory (its own float4 per
        // lobe: conflict-free), so the loops need no unrolling over lobes and no registers
        float4(*sg4)[8] = s_sg[wib][g];
        // lobe-outer: each lobe's S row is read once and used for the lane's 4 slices
#pragma unroll 1
        for (int c = 0; c < nmax; c++) {
            float2 s01 = make_float2(0.0f, 0.0f), s23 = s01, s45 = s01;
            if (valid && c < n) {
                const float2* sr = reinterpret_cast<const float2*>(Sg[c]);
                s01 = sr[0];
                s23 = sr[1];
                s45 = sr[2];
            }
            float sq[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                float qq = cf[q][0].x * s01.x;
                qq = qq + cf[q][0].y * s01.y;
                qq = qq + cf[q][1].x * s23.x;
                qq = qq + cf[q][1].y * s23.y;
                qq = qq + cf[q][2].x * s45.x;
                qq = qq + cf[q][2].y * s45.y;
                sq[q] = sqrtf(pmax(qq, 0.0f));
            }
            sg4[c][l] = make_float4(sq[0], sq[1], sq[2], sq[3]);
        }
        __syncwarp();
        // pairs t = 8b + (s ^ l) in slot s of lane l; lane l ends with pair 8b + l
        const int npq = nmax * (nmax - 1) / 2;
#pragma unroll 1
        for (int b = 0; b < npq; b += 8) {
            float v[8];
#pragma unroll
            for (int s = 0; s < 8; s++) {
                const int pr = s_pair[b + (s ^ l)];
                const float4 vi = sg4[pr >> 8][l], vj = sg4[pr & 0xff][l];
                const float ai[4] = {vi.x, vi.y, vi.z, vi.w}, aj[4] = {vj.x, vj.y, vj.z, vj.w};
                v[s] = part4(ai, aj);
            }
            const float s2 = group_sum8x8(v);
            const int t = b + l;
            if (t < npq) D[t] = (valid && (s_pair[t] & 0xff) < n) ? s2 : __uint_as_float(INF_BITS);
        }
        __syncwarp();
        unsigned alive = (1u << n) - 1u;
        const int np = nmax * (nmax - 1) / 2;
        for (int m = nmax; m > K; m--) {
            const bool act = valid && __popc(alive) > K;
            // lexicographic argmin (d, i, j) (D18) in two group reductions: the minimum d
            // (distances are finite and >= 0, dead pairs +inf), then the least (i << 8 | j)
            // among the pairs that attain it
            float dr[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const int t = l + 8 * r;
                dr[r] = t < np ? D[t] : __uint_as_float(INF_BITS);
            }
            float dmin = fminf(fminf(dr[0], dr[1]), fminf(dr[2], dr[3]));
#pragma unroll
            for (int o = 4; o >= 1; o >>= 1) dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
            unsigned code = 0xffffu;
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const int t = l + 8 * r;
                if (t < np && dr[r] == dmin) code = min(code, (unsigned)s_pair[t]);
            }
#pragma unroll
            for (int o = 4; o >= 1; o >>= 1) code = min(code, __shfl_xor_sync(0xffffffffu, code, o));
            const int bi = (int)(code >> 8), bj = (int)(code & 0xff);
            if (act && l < 7) lobe[bi][l] += lobe[bj][l];   // exact moment merge (D15)
            __syncwarp();
            if (m == K + 1) {   // the last merge: nothing reads sigma or D afterwards
                if (act) alive &= ~(1u << bj);
                break;
            }
            if (act && l < 6) Sg[bi][l] = deq32(lobe[bi][1 + l]) / deq32(lobe[bi][0]);
            __syncwarp();
            float sn[4];
            float2 m01 = make_float2(0.0f, 0.0f), m23 = m01, m45 = m01;
            if (act) {
                const float2* sr = reinterpret_cast<const float2*>(Sg[bi]);
                m01 = sr[0];
                m23 = sr[1];
                m45 = sr[2];
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                float qq = cf[q][0].x * m01.x;
                qq = qq + cf[q][0].y * m01.y;
                qq = qq + cf[q][1].x * m23.x;
                qq = qq + cf[q][1].y * m23.y;
                qq = qq + cf[q][2].x * m45.x;
                qq = qq + cf[q][2].y * m45.y;
                sn[q] = sqrtf(pmax(qq, 0.0f));
            }
            if (act) sg4[bi][l] = make_float4(sn[0], sn[1], sn[2], sn[3]);
            if (act) alive &= ~(1u << bj);
            __syncwarp();
            // d(bi, x) for x = 0..7 at once: slot s of lane l holds x = s ^ l (rows >= n are
            // never used: their sums land only in lanes >= n)
            float v[8];
#pragma unroll
            for (int s = 0; s < 8; s++) {
                const float4 vx = sg4[s ^ l][l];
                const float ax[4] = {vx.x, vx.y, vx.z, vx.w};
                v[s] = part4(sn, ax);
            }
            const float mine = group_sum8x8(v);
            if (act && l < n) {
                if (l != bi && ((alive >> l) & 1u)) D[l < bi ? pair_t(l, bi) : pair_t(bi, l)] = mine;
                if (l != bj) D[l < bj ? pair_t(l, bj) : pair_t(bj, l)] = __uint_as_float(INF_BITS);
            }
            __syncwarp();
        }
        if (valid) {
            // hard parents keep exactly K lobes: the set bits of alive, in list order
            unsigned a = alive;
#pragma unroll
            for (int slot = 0; slot < K; slot++) {
                const int c = __ffs(a) - 1;
                a &= a - 1u;
                if (l < 7) pclacc[((uint64_t)p * K + slot) * 7 + l] = lobe[c][l];
            }
            if (l == 0) pncl[p] = (uint8_t)K;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- SGGX-H, n > 16 (one warp per parent)
// d(i,j) tree for 32 slices held one per lane, for 32 pairs at once ("transpose-reduce"):
// lane p ends with the sum for pair p. At step h a lane keeps the half of its vector whose
// pair index has bit h equal to its own and adds the partner's partial; the partial sums it
// adds are s[l] and s[l+h] of the pinned tree (PREDICATES §9), so the result is bit-identical
// to the sequential tree (fp32 addition is commutative).
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int q = 0; q < h; q++) {
            const float send = up ? v[q] : v[q + h];
            const float keep = up ? v[q + h] : v[q];
            v[q] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
    return v[0];
}

// d(i, j) of two 32-slice sigma rows (float4 reads), the pinned tree in registers (PREDICATES §9)
__device__ __forceinline__ float dist_row(const float* ri, const float* rj) {
    const float4* a = reinterpret_cast<const float4*>(ri);
    const float4* b = reinterpret_cast<const float4*>(rj);
    float sv[32];
#pragma unroll
    for (int k4 = 0; k4 < 8; k4++) {
        const float4 u = a[k4], w = b[k4];
        sv[4 * k4 + 0] = fabsf(u.x - w.x);
        sv[4 * k4 + 1] = fabsf(u.y - w.y);
        sv[4 * k4 + 2] = fabsf(u.z - w.z);
        sv[4 * k4 + 3] = fabsf(u.w - w.w);
    }
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1)
#pragma unroll
        for (int q = 0; q < h; q++) sv[q] = sv[q] + sv[q + h];
    return sv[0];
}

constexpr int LOD_WARPS = 4;
constexpr int SIG_STRIDE = 36;   // sigma rows (16-byte aligned): 8 distinct rows per LDS.128 wavefront

template <int K>
struct LodSmem {
    static constexpr int MAXN = 8 * K;
    static constexpr int MAXP = MAXN * (MAXN - 1) / 2;
    static constexpr size_t list_bytes = MAXN * 7 * sizeof(long long);
    static constexpr size_t S_bytes = ((MAXN * 6 * sizeof(float) + 15) / 16) * 16;
    static constexpr size_t sig_bytes = MAXN * SIG_STRIDE * sizeof(float);
    static constexpr size_t D_bytes = ((MAXP * sizeof(unsigned long long) + 15) / 16) * 16;
    static constexpr size_t per_warp = list_bytes + S_bytes + sig_bytes + D_bytes;
    static constexpr size_t pairs_bytes = ((MAXP * sizeof(uint16_t) + 15) / 16) * 16;
    static constexpr size_t total = pairs_bytes + LOD_WARPS * per_warp;
};

template <int K>
__global__ void __launch_bounds__(LOD_WARPS * 32)
k_sggxh_warp(const uint32_t* __restrict__ list, const unsigned* __restrict__ counts,
             const uint8_t* __restrict__ cncl, const long long* __restrict__ cclacc,
             const uint32_t* __restrict__ start, uint8_t* __restrict__ pncl, long long* __restrict__ pclacc) {
    using SM = LodSmem<K>;
    constexpr int MAXP = SM::MAXP;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t* ptab = reinterpret_cast<uint16_t*>(smem_raw);   // t -> (i << 8) | j
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < MAXP; t += blockDim.x) {
        int j = 1;
        while ((j + 1) * j / 2 <= t) j++;
        ptab[t] = (uint16_t)(((t - j * (j - 1) / 2) << 8) | j);
    }
    __syncthreads();
    unsigned char* base = smem_raw + SM::pairs_bytes + wib * SM::per_warp;
    long long(*list_)[7] = reinterpret_cast<long long(*)[7]>(base);
    float(*Sm)[6] = reinterpret_cast<float(*)[6]>(base + SM::list_bytes);
    float(*sig)[SIG_STRIDE] = reinterpret_cast<float(*)[SIG_STRIDE]>(base + SM::list_bytes + SM::S_bytes);
    // D[t] = (bits of d << 32) | (i << 8 | j): one 64-bit compare orders by (d, i, j) (D18)
    unsigned long long* D = reinterpret_cast<unsigned long long*>(base + SM::list_bytes + SM::S_bytes + SM::sig_bytes);
    float cf[6];
#pragma unroll
    for (int e = 0; e < 6; e++) cf[e] = c_coef[lane][e];
    const unsigned lo = counts[1], hi = counts[2];
    for (unsigned w = lo + blockIdx.x * LOD_WARPS + wib; w < hi; w += gridDim.x * LOD_WARPS) {
        const uint64_t p = list[w];
        // dendrogram leaves in child-slot order, w = 0 dropped (D17)
        // one lane per (child, lobe slot): a single round of loads, compacted by ballot
        const int n = gather_lobes<K>(start, cncl, cclacc, p, lane, 0xffffffffu, &list_[0][0]);
        __syncwarp();
        unsigned long long alive = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
        // ---- S = M / w per lobe (one lane per lobe), sigma_k per lobe (one lane per slice)
        for (int c = lane; c < n; c += 32) {
            const float wf = deq32(list_[c][0]);
#pragma unroll
            for (int e = 0; e < 6; e++) Sm[c][e] = deq32(list_[c][1 + e]) / wf;
        }
        __syncwarp();
        const int np = n * (n - 1) / 2;
        for (int c = 0; c < n; c++) {
            float q = cf[0] * Sm[c][0];
#pragma unroll
            for (int e = 1; e < 6; e++) q = q + cf[e] * Sm[c][e];
            sig[c][lane] = sqrtf(pmax(q, 0.0f));
        }
        __syncwarp();
        // ---- initial distance matrix: one pair per lane, the pinned tree evaluated in
        // registers from two 32-slice sigma rows read as float4 (PREDICATES §9)
        for (int t = lane; t < np; t += 32) {
            const int pr = ptab[t];
            const float d = dist_row(sig[pr >> 8], sig[pr & 0xff]);
            D[t] = ((unsigned long long)__float_as_uint(d) << 32) | (unsigned)pr;
        }
        __syncwarp();
        // ---- SGGX-H merges: argmin of d over i < j, first in row-major order (D18)
        for (int m = n; m > K; m--) {
            unsigned long long best = ~0ull;
            for (int t = lane; t < np; t += 32) {
                const unsigned long long key = D[t];
                best = key < best ? key : best;
            }
            const unsigned bd = (unsigned)(best >> 32), bij = (unsigned)best;
            const unsigned dmin = __reduce_min_sync(0xffffffffu, bd);
            const unsigned ijmin = __reduce_min_sync(0xffffffffu, bd == dmin ? bij : 0xffffffffu);
            const int bi = (int)(ijmin >> 8), bj = (int)(ijmin & 0xff);
            if (lane < 7) list_[bi][lane] += list_[bj][lane];   // exact moment merge (D15)
            alive &= ~(1ull << bj);
            __syncwarp();
            if (m == K + 1) break;   // the last merge: nothing reads sigma or D afterwards
            if (lane < 6) Sm[bi][lane] = deq32(list_[bi][1 + lane]) / deq32(list_[bi][0]);
            __syncwarp();
            {
                float q = cf[0] * Sm[bi][0];
#pragma unroll
                for (int e = 1; e < 6; e++) q = q + cf[e] * Sm[bi][e];
                sig[bi][lane] = sqrtf(pmax(q, 0.0f));
            }
            __syncwarp();
            // new row d(bi, x): one pair per lane (the merged row is a broadcast read)
            for (int x = lane; x < n; x += 32) {
                if (x == bi || !((alive >> x) & 1ull)) continue;
                const float d = dist_row(sig[bi], sig[x]);
                const int a2 = x < bi ? x : bi, b2 = x < bi ? bi : x;
                D[pair_t(a2, b2)] = ((unsigned long long)__float_as_uint(d) << 32) | (unsigned)((a2 << 8) | b2);
            }
            // retire every pair of bj
            for (int x = lane; x < n; x += 32)
                if (x != bj) {
                    const int a = x < bj ? x : bj, b2 = x < bj ? bj : x;
                    D[pair_t(a, b2)] = ((unsigned long long)INF_BITS << 32) | (unsigned)((a << 8) | b2);
                }
            __syncwarp();
        }
        // output: surviving lobes in list order (K slots exactly, since n > K)
        unsigned long long a = alive;
#pragma unroll
        for (int slot = 0; slot < K; slot++) {
            const int cc = __ffsll((long long)a) - 1;
            a &= a - 1ull;
            if (lane < 7) pclacc[(p * K + slot) * 7 + lane] = list_[cc][lane];
        }
        if (lane == 0) pncl[p] = (uint8_t)K;
        __syncwarp();
    }
}

// ---------------------------------------------------------------- SGGX-H, 9 <= n <= 16 (half warp per parent)
// Two parents per warp, sixteen lanes each: the warp kernel's scheme at half width. Lane l
// computes sigma for slices l and l+16; distances are one pair per lane from float4-read
// sigma rows (dist_row, the pinned tree in registers); the argmin is a 16-lane xor reduce of
// the packed (d, i, j) keys. Both halves run max(n) merge steps, a half with fewer lobes
// idling through the surplus ones (bucket order makes the two n nearly always equal).
constexpr int HALF_WARPS = 4;
struct HalfPar {
    long long lobe[16][7];
    float S[16][6];
    float sig[16][SIG_STRIDE];
    unsigned long long D[120];
};

template <int K>
__global__ void __launch_bounds__(HALF_WARPS * 32)
k_sggxh_half(const uint32_t* __restrict__ list, const unsigned* __restrict__ counts,
             const uint8_t* __restrict__ cncl, const long long* __restrict__ cclacc,
             const uint32_t* __restrict__ start, uint8_t* __restrict__ pncl, long long* __restrict__ pclacc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t* ptab = reinterpret_cast<uint16_t*>(smem_raw);   // t -> (i << 8) | j, 120 entries
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane >> 4, l = lane & 15;
    for (int t = threadIdx.x; t < 120; t += blockDim.x) {
        int j = 1;
        while ((j + 1) * j / 2 <= t) j++;
        ptab[t] = (uint16_t)(((t - j * (j - 1) / 2) << 8) | j);
    }
    __syncthreads();
    HalfPar& H = reinterpret_cast<HalfPar*>(smem_raw + 256)[2 * wib + g];
    float cfa[6], cfb[6];
#pragma unroll
    for (int e = 0; e < 6; e++) {
        cfa[e] = c_coef[l][e];
        cfb[e] = c_coef[l + 16][e];
    }
    const unsigned lo = counts[0], hi = counts[1];
    for (unsigned u = blockIdx.x * HALF_WARPS + wib; lo + 2 * u < hi; u += gridDim.x * HALF_WARPS) {
        const unsigned idx = lo + 2 * u + g;
        const bool valid = idx < hi;
        const uint64_t p = valid ? list[idx] : 0;
        uint32_t c0 = 0, c1 = 0;
        if (valid) {
            c0 = start[p];
            c1 = start[p + 1];
        }
        // dendrogram leaves in child-slot order, w = 0 dropped (D17): rounds of 16 slots
        const int slots = (int)(c1 - c0) * K;
        int n = 0;
        for (int b = 0; b < 8 * K; b += 16) {
            const int sl = b + l;
            bool has = false;
            const long long* src = nullptr;
            if (sl < slots) {
                const uint64_t x = c0 + sl / K;
                const int q = sl % K;
                src = cclacc + (x * K + q) * 7;
                has = q < cncl[x] && src[0] != 0;
            }
            const unsigned bal = (__ballot_sync(0xffffffffu, has) >> (16 * g)) & 0xffffu;
            if (has) {
                const int c = n + __popc(bal & ((1u << l) - 1u));
                VOX_DCHECK(c < 16, 5);
#pragma unroll
                for (int e = 0; e < 7; e++) H.lobe[c][e] = src[e];
            }
            n += __popc(bal);
        }
        __syncwarp();
        const int nmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
        unsigned alive = (1u << n) - 1u;
        if (l < n) {
            const float wf = deq32(H.lobe[l][0]);
#pragma unroll
            for (int e = 0; e < 6; e++) H.S[l][e] = deq32(H.lobe[l][1 + e]) / wf;
        }
        __syncwarp();
        for (int c = 0; c < nmax; c++) {
            if (c < n) {
                float qa = cfa[0] * H.S[c][0], qb = cfb[0] * H.S[c][0];
#pragma unroll
                for (int e = 1; e < 6; e++) {
                    qa = qa + cfa[e] * H.S[c][e];
                    qb = qb + cfb[e] * H.S[c][e];
                }
                H.sig[c][l] = sqrtf(pmax(qa, 0.0f));
                H.sig[c][l + 16] = sqrtf(pmax(qb, 0.0f));
            }
        }
        __syncwarp();
        const int np = n * (n - 1) / 2, npmax = nmax * (nmax - 1) / 2;
        for (int t = l; t < npmax; t += 16) {
            if (t < np) {
                const int pr = ptab[t];
                const float d = dist_row(H.sig[pr >> 8], H.sig[pr & 0xff]);
                H.D[t] = ((unsigned long long)__float_as_uint(d) << 32) | (unsigned)pr;
            }
        }
        __syncwarp();
        // ---- SGGX-H merges: argmin of d over i < j, first in row-major order (D18)
        for (int m = nmax; m > K; m--) {
            const bool act = m <= n;
            unsigned long long best = ~0ull;
            for (int t = l; t < npmax; t += 16) {
                if (t < np) {
                    const unsigned long long key = H.D[t];
                    best = key < best ? key : best;
                }
            }
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) {
                const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
                best = y < best ? y : best;
            }
            const int bi = (int)((best >> 8) & 0xff), bj = (int)(best & 0xff);
            if (act && l < 7) H.lobe[bi][l] += H.lobe[bj][l];   // exact moment merge (D15)
            if (act) alive &= ~(1u << bj);
            __syncwarp();
            if (m == K + 1) break;   // the last merge: nothing reads sigma or D afterwards
            if (act && l < 6) H.S[bi][l] = deq32(H.lobe[bi][1 + l]) / deq32(H.lobe[bi][0]);
            __syncwarp();
            if (act) {
                float qa = cfa[0] * H.S[bi][0], qb = cfb[0] * H.S[bi][0];
#pragma unroll
                for (int e = 1; e < 6; e++) {
                    qa = qa + cfa[e] * H.S[bi][e];
                    qb = qb + cfb[e] * H.S[bi][e];
                }
                H.sig[bi][l] = sqrtf(pmax(qa, 0.0f));
                H.sig[bi][l + 16] = sqrtf(pmax(qb, 0.0f));
            }
            __syncwarp();
            const int x = l;
            if (act && x < n) {
                if (x != bi && ((alive >> x) & 1u)) {   // new row d(bi, x)
                    const float d = dist_row(H.sig[bi], H.sig[x]);
                    const int a2 = x < bi ? x : bi, b2 = x < bi ? bi : x;
                    H.D[pair_t(a2, b2)] = ((unsigned long long)__float_as_uint(d) << 32) | (unsigned)((a2 << 8) | b2);
                }
                if (x != bj) {                            // retire every pair of bj
                    const int a = x < bj ? x : bj, b2 = x < bj ? bj : x;
                    H.D[pair_t(a, b2)] = ((unsigned long long)INF_BITS << 32) | (unsigned)((a << 8) | b2);
                }
            }
            __syncwarp();
        }
        // output: surviving lobes in list order (K slots exactly, since n > K)
        if (valid) {
            unsigned a = alive;
#pragma unroll
            for (int slot = 0; slot < K; slot++) {
                const int cc = __ffs(a) - 1;
                a &= a - 1u;
                if (l < 7) pclacc[(p * K + slot) * 7 + l] = H.lobe[cc][l];
            }
            if (l == 0) pncl[p] = (uint8_t)K;
        }
        __syncwarp();
    }
}

// fp32 views from the exact accumulators (§8: one rounding of the fixed-point sum): a word per
// thread, grid-stride, so every array is read and written coalesced. Lobes past ncl are 0.
__global__ void k_finalize(uint64_t n, const long long* __restrict__ acc, float* __restrict__ mass,
                           float* __restrict__ m6, const uint8_t* __restrict__ ncl, const long long* __restrict__ clacc,
                           float* __restrict__ cl, int K) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (mass)
        for (uint64_t v = t0; v < n; v += stride) mass[v] = deq32(acc[7 * v]);
    if (m6)
        for (uint64_t w = t0; w < 6 * n; w += stride) {
            const uint64_t v = w / 6;
            m6[w] = deq32(acc[7 * v + 1 + (w - 6 * v)]);
        }
    if (cl) {
        const uint64_t per = 7ull * K;
        for (uint64_t w = t0; w < per * n; w += stride) {
            const uint64_t v = w / per;
            const int q = (int)((w - per * v) / 7);
            cl[w] = q < ncl[v] ? deq32(clacc[w]) : 0.0f;
        }
    }
}

static unsigned grid_for(uint64_t n, int threads = 256) {
    uint64_t b = (n + threads - 1) / threads;
    if (b > 148ull * 32) b = 148ull * 32;
    if (b == 0) b = 1;
    return (unsigned)b;
}

cudaError_t launch_finalize(vox_ctx* c, cudaStream_t s, uint64_t n, const long long* acc, const uint8_t* ncl,
                            const long long* clacc, float* mass, float* m6, float* cl) {
    if (n == 0 || (!mass && !m6 && !cl)) return cudaSuccess;
    k_finalize<<<grid_for(6 * n), 256, 0, s>>>(n, acc, mass, m6, ncl, clacc, cl, (int)c->K);
    c->st.launches++;
    return cudaGetLastError();
}


#define CK(x)                                                          \
    do {                                                               \
        cudaError_t e_ = (x);                                          \
        if (e_ != cudaSuccess) {                                       \
            c->err = std::string(#x) + ": " + cudaGetErrorString(e_);  \
            return e_ == cudaErrorMemoryAllocation ? VOX_ERR_OOM : VOX_ERR_CUDA; \
        }                                                              \
    } while (0)

vox_status ensure_f32(vox_ctx* c, int level) {
    Level& L = c->lv[level];
    if (L.f32 || L.n == 0) return VOX_OK;
    CK(dalloc(c, (void**)&L.mass, L.n * 4));
    CK(dalloc(c, (void**)&L.m6, L.n * 24));
    if (level > 0) CK(dalloc(c, (void**)&L.cl, L.n * c->K * 28));
    CK(launch_finalize(c, c->stream, L.n, L.acc, L.ncl, L.clacc, L.mass, L.m6, level > 0 ? L.cl : nullptr));
    L.f32 = true;
    return VOX_OK;
}

template <int K>
static vox_status run_level(vox_ctx* c, const Level& C, int leaf, const uint32_t* start, Level& P) {
    constexpr int MAXN = 8 * K;
    const uint64_t V = P.n;
    uint8_t* nlob = nullptr;
    unsigned *hist = nullptr, *cursor = nullptr, *counts = nullptr;
    uint32_t* list = nullptr;
    CK(dalloc(c, (void**)&nlob, V));
    CK(dalloc(c, (void**)&hist, 4 * (MAXN + 1) * 2 + 32));
    cursor = hist + (MAXN + 1);
    counts = cursor + (MAXN + 1);
    CK(dalloc(c, (void**)&list, V * 4));
    CK(cudaMemsetAsync(hist, 0, 4 * (MAXN + 1), c->stream));
    timer_begin(c, c->t_prep);
    if (leaf) {
        uint64_t pb = ((V + PREP_PAR - 1) / PREP_PAR + PREP_WARPS - 1) / PREP_WARPS;
        const size_t psm = (size_t)PREP_WARPS * (PREP_WARP_WORDS + PREP_PAR * K * 7) * sizeof(long long);
        CK(cudaFuncSetAttribute(k_lod_prep_leaf<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
        // resident blocks per SM (shared memory bound), once per K (thread-safe static init)
        static const int occ = [psm]() {
            int o = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_lod_prep_leaf<K>, PREP_WARPS * 32, psm) !=
                cudaSuccess) {
                cudaGetLastError();
                o = 3;
            }
            return o < 1 ? 1 : o;
        }();
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->dev);
        pb = std::min<uint64_t>(std::max<uint64_t>(pb, 1), (uint64_t)nsm * occ);
        k_lod_prep_leaf<K><<<(unsigned)pb, PREP_WARPS * 32, psm, c->stream>>>(C.acc, start, V, P.acc, P.ncl,
                                                                            P.clacc, nlob, hist);
    } else {
        k_lod_prep<K><<<grid_for(V), 256, 0, c->stream>>>(C.acc, C.ncl, C.clacc, leaf, start, V, P.acc, P.ncl,
                                                         P.clacc, nlob, hist);
    }
    timer_end(c, c->t_prep);
    // key, mass and m6 of the level are final here (SGGX-H only writes lobes): an event lets
    // vox_copy_level_async start their D2H while the clustering runs
    {
        const int l = (int)(&P - c->lv);
        if (!c->ev_level[l]) CK(cudaEventCreateWithFlags(&c->ev_level[l], cudaEventDisableTiming));
        CK(cudaEventRecord(c->ev_level[l], c->stream));
        c->ev_level_ok[l] = true;
    }
    k_bucket_init<<<1, 32, 0, c->stream>>>(hist, K, MAXN, cursor, counts, c->d_lodwork);
    const uint64_t sb = (V + 256ull * SCATTER_PER_THREAD - 1) / (256ull * SCATTER_PER_THREAD);
    k_bucket_scatter<<<(unsigned)(sb ? sb : 1), 256, 0, c->stream>>>(nlob, V, K, MAXN, cursor, list);
    c->st.launches += 3;
    // grids cover the worst case (every parent hard); blocks stride over the actual counts
    if (c->dmode == 1) {   // histogram distance (§10): one kernel for every n > K
        timer_begin(c, c->t_warp);
        CK(launch_sggxh_hist(c, K, list, counts, C, leaf, start, P));
        timer_end(c, c->t_warp);
        c->st.launches++;
    } else {
    if (K < 8) {
        uint64_t qb = ((V + 3) / 4 + QUAD_WARPS - 1) / QUAD_WARPS;
        qb = std::min<uint64_t>(std::max<uint64_t>(qb, 1), 148ull * 48);
        timer_begin(c, c->t_quad);
        k_sggxh_quad<K><<<(unsigned)qb, QUAD_WARPS * 32, 0, c->stream>>>(list, counts, C.acc, C.ncl, C.clacc, leaf,
                                                                        start, P.ncl, P.clacc);
        timer_end(c, c->t_quad);
        c->st.launches++;
    }
    if (!leaf && MAXN > 8) {
        const size_t smem = 256 + 2 * HALF_WARPS * sizeof(HalfPar);
        CK(cudaFuncSetAttribute(k_sggxh_half<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        uint64_t hb = ((V + 1) / 2 + HALF_WARPS - 1) / HALF_WARPS;
        hb = std::min<uint64_t>(std::max<uint64_t>(hb, 1), 148ull * 32);
        timer_begin(c, c->t_half);
        k_sggxh_half<K><<<(unsigned)hb, HALF_WARPS * 32, smem, c->stream>>>(list, counts, C.ncl, C.clacc, start,
                                                                           P.ncl, P.clacc);
        timer_end(c, c->t_half);
        c->st.launches++;
    }
    if (!leaf && MAXN > 16) {
        const size_t smem = LodSmem<K>::total;
        CK(cudaFuncSetAttribute(k_sggxh_warp<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        uint64_t wb = (V + LOD_WARPS - 1) / LOD_WARPS;
        wb = std::min<uint64_t>(std::max<uint64_t>(wb, 1), 148ull * 32);
        timer_begin(c, c->t_warp);
        k_sggxh_warp<K><<<(unsigned)wb, LOD_WARPS * 32, smem, c->stream>>>(list, counts, C.ncl, C.clacc, start,
                                                                          P.ncl, P.clacc);
        timer_end(c, c->t_warp);
        c->st.launches++;
    }
    }
    CK(cudaGetLastError());
    dfree(c, list);
    dfree(c, hist);
    dfree(c, nlob);
    return VOX_OK;
}

vox_status build_level(vox_ctx* c, int l) {
    static const char* names[VOX_MAX_LEVELS] = {"level 0", "level 1", "level 2", "level 3", "level 4", "level 5", "level 6",
                                                "level 7", "level 8", "level 9", "level 10", "level 11", "level 12",
                                                "level 13"};
    VOX_RANGE(names[l < VOX_MAX_LEVELS ? l : 0]);
    Level& C = c->lv[l - 1];
    Level& P = c->lv[l];
    free_level(c, P);
    c->ev_level_ok[l] = false;
    const uint64_t n = C.n;
    const uint32_t K = c->K;
    if (n == 0) return VOX_OK;
    timer_begin(c, c->t_lodscan);
    // one single-pass scan (k_scan.cu): run-head flags computed from the child keys on the fly,
    // each head's parent start and key scattered by the scan's output -- no flag or count
    // arrays. start / P.key are sized by n >= V.
    uint32_t* start = nullptr;
    uint32_t* total = nullptr;
    CK(dalloc(c, (void**)&start, (n + 1) * 4));
    CK(dalloc(c, (void**)&P.key, n * 8));
    CK(dalloc(c, (void**)&total, 16));
    CK(scan_run_heads(c, C.key, n, start, P.key, total));
    uint32_t V = 0;
    CK(readback(c, {{&V, total, 4}}));
    dfree(c, total);
    timer_end(c, c->t_lodscan);
    P.n = V;
    CK(dalloc(c, (void**)&P.acc, (uint64_t)V * 56));
    CK(dalloc(c, (void**)&P.ncl, (uint64_t)V));
    CK(dalloc(c, (void**)&P.clacc, (uint64_t)V * K * 56));
    timer_begin(c, c->t_lod);
    const int leaf = (l == 1);
    vox_status s;
    switch (K) {
        case 1: s = run_level<1>(c, C, leaf, start, P); break;
        case 2: s = run_level<2>(c, C, leaf, start, P); break;
        case 3: s = run_level<3>(c, C, leaf, start, P); break;
        case 4: s = run_level<4>(c, C, leaf, start, P); break;
        case 5: s = run_level<5>(c, C, leaf, start, P); break;
        case 6: s = run_level<6>(c, C, leaf, start, P); break;
        case 7: s = run_level<7>(c, C, leaf, start, P); break;
        default: s = run_level<8>(c, C, leaf, start, P); break;
    }
    timer_end(c, c->t_lod);
    dfree(c, start);
    return s;
}

// ---------------------------------------------------------------- multi-GPU level records

uint64_t record_bytes(uint32_t K) { return 72 + 56ull * K; }

__global__ void k_pack(uint64_t n, const uint64_t* __restrict__ key, const long long* __restrict__ acc,
                       const uint8_t* __restrict__ ncl, const long long* __restrict__ clacc, int K, int leaf,
                       long long* __restrict__ out) {
    const uint64_t words = 9 + 7ull * K;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        long long* r = out + v * words;
        r[0] = (long long)key[v];
        for (int e = 0; e < 7; e++) r[1 + e] = acc[7 * v + e];
        const int m = leaf ? (acc[7 * v] > 0) : ncl[v];
        r[8] = m;
        for (int q = 0; q < K; q++)   // lobe slots >= ncl hold no data in the level: exported as 0
            for (int e = 0; e < 7; e++)
                r[9 + 7 * q + e] = q < m ? (leaf ? acc[7 * v + e] : clacc[(v * K + q) * 7 + e]) : 0;
    }
}

__global__ void k_unpack(uint64_t n, const long long* __restrict__ in, int K, uint64_t* __restrict__ key,
                         long long* __restrict__ acc, uint8_t* __restrict__ ncl, long long* __restrict__ clacc,
                         unsigned* __restrict__ flags) {
    const uint64_t words = 9 + 7ull * K;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const long long* r = in + v * words;
        key[v] = (uint64_t)r[0];
        if (v > 0 && (uint64_t)in[(v - 1) * words] >= (uint64_t)r[0]) atomicOr(flags, 1u);
        if (r[8] < 0 || r[8] > K) atomicOr(flags, 1u);
        for (int e = 0; e < 7; e++) acc[7 * v + e] = r[1 + e];
        ncl[v] = (uint8_t)r[8];
        for (int q = 0; q < K; q++)
            for (int e = 0; e < 7; e++) clacc[(v * K + q) * 7 + e] = r[9 + 7 * q + e];
    }
}

cudaError_t launch_pack(vox_ctx* c, int level, void* buf) {
    Level& L = c->lv[level];
    if (L.n == 0) return cudaSuccess;
    k_pack<<<grid_for(L.n), 256, 0, c->stream>>>(L.n, L.key, L.acc, L.ncl, L.clacc, (int)c->K, level == 0,
                                                 (long long*)buf);
    c->st.launches++;
    return cudaGetLastError();
}

vox_status unpack_level(vox_ctx* c, int level, const void* buf, uint64_t n) {
    Level& L = c->lv[level];
    free_level(c, L);
    L.n = n;
    const uint32_t K = c->K;
    if (n == 0) return VOX_OK;
    CK(dalloc(c, (void**)&L.key, n * 8));
    CK(dalloc(c, (void**)&L.acc, n * 56));
    CK(dalloc(c, (void**)&L.ncl, n));
    CK(dalloc(c, (void**)&L.clacc, n * K * 56));
    CK(cudaMemsetAsync(c->d_flags, 0, 4, c->stream));
    k_unpack<<<grid_for(n), 256, 0, c->stream>>>(n, (const long long*)buf, (int)K, L.key, L.acc, L.ncl, L.clacc,
                                                 c->d_flags);
    c->st.launches++;
    unsigned fl = 0;
    CK(readback(c, {{&fl, c->d_flags, 4}}));
    if (fl) {
        c->err = "import: records not strictly ascending or bad lobe count";
        free_level(c, L);
        return VOX_ERR_COMM;
    }
    return VOX_OK;
}

}  // namespace vox
