// k_lod.cu -- the 2x2x2 Morton pyramid with per-parent SGGX-H clustering
// (§4.4 Eq. similarity; docs/PREDICATES.md §9), fp32 finalisation of levels, and
// the fixed-size level records used by the multi-GPU gather.
//
// Parents are runs of equal key>>3 in the sorted child level (Morton order is hierarchical,
// so no re-sort). One warp per parent: lanes 0..6 sum the 7 accumulators exactly; the
// children's lobes are gathered into shared memory; if more than K remain, SGGX-H runs with
// lane = slice for sigma (32 slices = 32 lanes) and lane = pair for distances and argmin.
#include <cub/cub.cuh>

#include <cmath>

#include "vox_internal.cuh"

namespace vox {

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

// sigma_k of a lobe given by its 7 accumulators (w, M6)
__device__ __forceinline__ float lobe_sigma(const long long* a, int k) {
    const float wf = deq32(a[0]);
    float q = c_coef[k][0] * (deq32(a[1]) / wf);
#pragma unroll
    for (int e = 1; e < 6; e++) q = q + c_coef[k][e] * (deq32(a[1 + e]) / wf);
    return sqrtf(pmax(q, 0.0f));
}

// d(i,j): |sigma_i - sigma_j| summed in the fixed xor-butterfly tree order (PREDICATES §9)
__device__ __forceinline__ float lobe_dist(const float* si, const float* sj) {
    float s[32];
#pragma unroll
    for (int k = 0; k < 32; k++) s[k] = fabsf(si[k] - sj[k]);
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1)
#pragma unroll
        for (int l = 0; l < h; l++) s[l] = s[l] + s[l + h];
    return s[0];
}

constexpr int LOD_WARPS = 4;
constexpr int SIG_STRIDE = 33;   // padded sigma rows: lanes reading distinct rows hit distinct banks

template <int K>
struct LodSmem {
    static constexpr int MAXN = 8 * K;
    static constexpr size_t list_bytes = MAXN * 7 * sizeof(long long);
    static constexpr size_t sig_bytes = MAXN * SIG_STRIDE * sizeof(float);
    static constexpr size_t dist_bytes = MAXN * MAXN * sizeof(float);
    static constexpr size_t per_warp = list_bytes + sig_bytes + dist_bytes;
};

template <int K>
__global__ void __launch_bounds__(LOD_WARPS * 32)
k_pyramid(const uint64_t* __restrict__ ckey, const long long* __restrict__ cacc, const uint8_t* __restrict__ cncl,
          const long long* __restrict__ cclacc, int child_is_leaf, const uint32_t* __restrict__ start, uint64_t V,
          uint64_t* __restrict__ pkey, long long* __restrict__ pacc, uint8_t* __restrict__ pncl,
          long long* __restrict__ pclacc) {
    using SM = LodSmem<K>;
    constexpr int MAXN = SM::MAXN;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* base = smem_raw + wib * SM::per_warp;
    long long(*list)[7] = reinterpret_cast<long long(*)[7]>(base);
    float(*sig)[SIG_STRIDE] = reinterpret_cast<float(*)[SIG_STRIDE]>(base + SM::list_bytes);
    float(*dist)[MAXN] = reinterpret_cast<float(*)[MAXN]>(base + SM::list_bytes + SM::sig_bytes);

    for (uint64_t p = blockIdx.x * (uint64_t)LOD_WARPS + wib; p < V; p += (uint64_t)gridDim.x * LOD_WARPS) {
        const uint32_t c0 = start[p], c1 = start[p + 1];
        const int nch = (int)(c1 - c0);
        // naive aggregate: exact sums of the children's accumulators
        if (lane < 7) {
            long long s = 0;
            for (uint32_t x = c0; x < c1; x++) s += cacc[7 * (uint64_t)x + lane];
            pacc[7 * p + lane] = s;
        }
        if (lane == 0) pkey[p] = ckey[c0] >> 3;
        // dendrogram leaves: the children's lobes in child-slot order, w = 0 dropped (D17)
        int cnt = 0;
        if (lane < nch) {
            const uint64_t x = c0 + lane;
            if (child_is_leaf) cnt = cacc[7 * x] > 0;
            else
                for (int q = 0; q < cncl[x]; q++) cnt += cclacc[(x * K + q) * 7] != 0;
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int n = __shfl_sync(0xffffffffu, incl, 7);
        if (lane < nch && cnt) {
            const uint64_t x = c0 + lane;
            int o = incl - cnt;
            if (child_is_leaf) {
                for (int e = 0; e < 7; e++) list[o][e] = cacc[7 * x + e];
            } else {
                for (int q = 0; q < cncl[x]; q++) {
                    const long long* src = cclacc + (x * K + q) * 7;
                    if (src[0] == 0) continue;
                    for (int e = 0; e < 7; e++) list[o][e] = src[e];
                    o++;
                }
            }
        }
        __syncwarp();
        unsigned long long alive = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
        if (n > K) {
            // SGGX-H: merge the closest pair until K lobes remain
            for (int cc = 0; cc < n; cc++) sig[cc][lane] = lobe_sigma(list[cc], lane);
            __syncwarp();
            for (int i = 0; i + 1 < n; i++)
                for (int j = i + 1 + lane; j < n; j += 32) dist[i][j] = lobe_dist(sig[i], sig[j]);
            __syncwarp();
            for (int m = n; m > K; m--) {
                // first minimum of d over i < j in row-major order (D18): lexicographic (d, i, j)
                unsigned long long best = ~0ull;
                for (int i = 0; i + 1 < n; i++) {
                    if (!((alive >> i) & 1ull)) continue;
                    for (int j = i + 1 + lane; j < n; j += 32) {
                        if (!((alive >> j) & 1ull)) continue;
                        const unsigned long long key =
                            ((unsigned long long)__float_as_uint(dist[i][j]) << 32) | (unsigned)(i << 8) | (unsigned)j;
                        best = key < best ? key : best;
                    }
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) {
                    const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
                    best = y < best ? y : best;
                }
                const int bi = (int)((best >> 8) & 0xff), bj = (int)(best & 0xff);
                if (lane < 7) list[bi][lane] += list[bj][lane];   // exact moment merge (D15)
                alive &= ~(1ull << bj);
                __syncwarp();
                sig[bi][lane] = lobe_sigma(list[bi], lane);
                __syncwarp();
                for (int x = lane; x < n; x += 32) {
                    if (x == bi || !((alive >> x) & 1ull)) continue;
                    const int a = x < bi ? x : bi, b = x < bi ? bi : x;
                    dist[a][b] = lobe_dist(sig[a], sig[b]);
                }
                __syncwarp();
            }
        }
        // output: surviving lobes in list order, zero-filled to K slots
        int slot = 0;
        for (int cc = 0; cc < n; cc++) {
            if (!((alive >> cc) & 1ull)) continue;
            if (lane < 7) pclacc[(p * K + slot) * 7 + lane] = list[cc][lane];
            slot++;
        }
        for (int q = slot; q < K; q++)
            if (lane < 7) pclacc[(p * K + q) * 7 + lane] = 0;
        if (lane == 0) pncl[p] = (uint8_t)slot;
        __syncwarp();
    }
}

__global__ void k_pheads(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ flags) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        flags[i] = (i == 0 || (keys[i] >> 3) != (keys[i - 1] >> 3)) ? 1u : 0u;
}

__global__ void k_pstarts(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ incl, uint64_t n,
                          uint32_t* __restrict__ start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (flags[i]) start[incl[i] - 1] = (uint32_t)i;
        if (i == n - 1) start[incl[i]] = (uint32_t)n;
    }
}

__global__ void k_finalize(uint64_t n, const long long* __restrict__ acc, float* __restrict__ mass,
                           float* __restrict__ m6, const uint8_t* __restrict__ ncl, const long long* __restrict__ clacc,
                           float* __restrict__ cl, int K) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        mass[v] = deq32(acc[7 * v]);
        for (int e = 0; e < 6; e++) m6[6 * v + e] = deq32(acc[7 * v + 1 + e]);
        if (cl) {
            const int m = ncl[v];
            for (int q = 0; q < K; q++)
                for (int e = 0; e < 7; e++)
                    cl[(v * K + q) * 7 + e] = q < m ? deq32(clacc[(v * K + q) * 7 + e]) : 0.0f;
        }
    }
}

static unsigned grid_for(uint64_t n, int threads = 256) {
    uint64_t b = (n + threads - 1) / threads;
    if (b > 148ull * 32) b = 148ull * 32;
    if (b == 0) b = 1;
    return (unsigned)b;
}

cudaError_t launch_finalize(vox_ctx* c, Level& L, bool clusters) {
    if (L.n == 0) return cudaSuccess;
    k_finalize<<<grid_for(L.n), 256, 0, c->stream>>>(L.n, L.acc, L.mass, L.m6, clusters ? L.ncl : nullptr,
                                                     clusters ? L.clacc : nullptr, clusters ? L.cl : nullptr,
                                                     (int)c->K);
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

template <int K>
static cudaError_t launch_pyramid(vox_ctx* c, const Level& C, int child_is_leaf, const uint32_t* start, Level& P) {
    const size_t smem = LodSmem<K>::per_warp * LOD_WARPS;
    cudaError_t e = cudaFuncSetAttribute(k_pyramid<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    uint64_t blocks = (P.n + LOD_WARPS - 1) / LOD_WARPS;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    k_pyramid<K><<<(unsigned)blocks, LOD_WARPS * 32, smem, c->stream>>>(C.key, C.acc, C.ncl, C.clacc, child_is_leaf,
                                                                       start, P.n, P.key, P.acc, P.ncl, P.clacc);
    c->st.launches++;
    return cudaGetLastError();
}

vox_status build_level(vox_ctx* c, int l) {
    Level& C = c->lv[l - 1];
    Level& P = c->lv[l];
    free_level(c, P);
    const uint64_t n = C.n;
    const uint32_t K = c->K;
    if (n == 0) return VOX_OK;
    timer_begin(c, c->t_lodscan);
    uint32_t *flags = nullptr, *incl = nullptr, *start = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    CK(dalloc(c, (void**)&flags, n * 4));
    CK(dalloc(c, (void**)&incl, n * 4));
    k_pheads<<<grid_for(n), 256, 0, c->stream>>>(C.key, n, flags);
    c->st.launches++;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, flags, incl, (int64_t)n, c->stream));
    CK(dalloc(c, &tmp, tb));
    CK(cub::DeviceScan::InclusiveSum(tmp, tb, flags, incl, (int64_t)n, c->stream));
    c->st.launches++;
    uint32_t V = 0;
    CK(cudaMemcpyAsync(&V, incl + n - 1, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(dalloc(c, (void**)&start, ((uint64_t)V + 1) * 4));
    k_pstarts<<<grid_for(n), 256, 0, c->stream>>>(flags, incl, n, start);
    c->st.launches++;
    dfree(c, tmp);
    dfree(c, incl);
    dfree(c, flags);
    timer_end(c, c->t_lodscan);
    P.n = V;
    CK(dalloc(c, (void**)&P.key, (uint64_t)V * 8));
    CK(dalloc(c, (void**)&P.acc, (uint64_t)V * 56));
    CK(dalloc(c, (void**)&P.mass, (uint64_t)V * 4));
    CK(dalloc(c, (void**)&P.m6, (uint64_t)V * 24));
    CK(dalloc(c, (void**)&P.ncl, (uint64_t)V));
    CK(dalloc(c, (void**)&P.clacc, (uint64_t)V * K * 56));
    CK(dalloc(c, (void**)&P.cl, (uint64_t)V * K * 28));
    timer_begin(c, c->t_lod);
    const int leaf = (l == 1);
    cudaError_t e;
    switch (K) {
        case 1: e = launch_pyramid<1>(c, C, leaf, start, P); break;
        case 2: e = launch_pyramid<2>(c, C, leaf, start, P); break;
        case 3: e = launch_pyramid<3>(c, C, leaf, start, P); break;
        case 4: e = launch_pyramid<4>(c, C, leaf, start, P); break;
        case 5: e = launch_pyramid<5>(c, C, leaf, start, P); break;
        case 6: e = launch_pyramid<6>(c, C, leaf, start, P); break;
        case 7: e = launch_pyramid<7>(c, C, leaf, start, P); break;
        default: e = launch_pyramid<8>(c, C, leaf, start, P); break;
    }
    CK(e);
    timer_end(c, c->t_lod);
    dfree(c, start);
    CK(launch_finalize(c, P, true));
    return VOX_OK;
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
        for (int q = 0; q < K; q++)
            for (int e = 0; e < 7; e++)
                r[9 + 7 * q + e] = leaf ? (q == 0 && m ? acc[7 * v + e] : 0) : clacc[(v * K + q) * 7 + e];
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
    CK(dalloc(c, (void**)&L.mass, n * 4));
    CK(dalloc(c, (void**)&L.m6, n * 24));
    CK(dalloc(c, (void**)&L.ncl, n));
    CK(dalloc(c, (void**)&L.clacc, n * K * 56));
    CK(dalloc(c, (void**)&L.cl, n * K * 28));
    CK(cudaMemsetAsync(c->d_flags, 0, 4, c->stream));
    k_unpack<<<grid_for(n), 256, 0, c->stream>>>(n, (const long long*)buf, (int)K, L.key, L.acc, L.ncl, L.clacc,
                                                 c->d_flags);
    c->st.launches++;
    unsigned fl = 0;
    CK(cudaMemcpyAsync(&fl, c->d_flags, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (fl) {
        c->err = "import: records not strictly ascending or bad lobe count";
        free_level(c, L);
        return VOX_ERR_COMM;
    }
    CK(launch_finalize(c, L, true));
    return VOX_OK;
}

}  // namespace vox
