// SGGX-H with the paper's histogram distance (distance_mode = 1; docs/PREDICATES.md §10,
// SURVEY §8(f) NEXT-1): N whole-sphere samples per SGGX, a 5x5x5 histogram
// (P:389), the sliced Wasserstein-1 distance between histograms over the 32 slices of
// §9, in exact integer arithmetic.
//
// One warp per parent with n > K (every level, leaves included). A lobe's histogram is built
// by the whole warp: lane l takes samples l, l+32, ... of the sample table (SoA in global,
// L1/L2-resident), bins them with the pinned fp32 sequence and counts into its own byte
// column of a [125][32] shared-memory counter block (no atomics: N <= 8160 keeps a lane's
// count <= 255); a dp4a pass sums the columns. A pair distance has lane k walk slice k's
// 124 sorted bins (tables transposed [r][32] in shared memory, conflict-free) accumulating
// |C| * gap in 64-bit integers; a xor-shuffle sum finishes it (exact, order-free).
#include "vox_internal.cuh"
#include "hist_cells.cuh"

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

namespace vox {

constexpr int HB = 125;   // histogram cells
constexpr int HR = 124;   // sorted gaps per slice

// ---------------------------------------------------------------- host tables (§10)
void host_hist_tables(int N, std::vector<float>& u, std::vector<uint8_t>& permT, std::vector<uint32_t>& gapT) {
    const double pi = 3.14159265358979323846;
    const double golden_angle = pi * (3.0 - std::sqrt(5.0));
    u.assign(3 * (size_t)N, 0.0f);
    for (int s = 0; s < N; s++) {
        const double z = 1.0 - (2.0 * s + 1.0) / N;
        const double rho = std::sqrt(1.0 - z * z);
        const double phi = s * golden_angle;
        u[s] = (float)(rho * std::cos(phi));
        u[N + s] = (float)(rho * std::sin(phi));
        u[2 * (size_t)N + s] = (float)z;
    }
    float theta[32][3], coef[32][6];
    host_theta(theta, coef);
    permT.assign(HR * 32, 0);
    gapT.assign(HR * 32, 0);
    for (int k = 0; k < 32; k++) {
        long long P[HB];
        int idx[HB];
        for (int b = 0; b < HB; b++) {
            const int b0 = b % 5, b1 = (b / 5) % 5, b2 = b / 25;
            double x = (double)theta[k][0] * (2 * b0 - 4) + (double)theta[k][1] * (2 * b1 - 4);
            x = x + (double)theta[k][2] * (2 * b2 - 4);
            P[b] = std::llrint(x * 65536.0);
            idx[b] = b;
        }
        std::stable_sort(idx, idx + HB, [&](int a, int b) { return P[a] < P[b]; });
        for (int r = 0; r < HR; r++) {
            permT[r * 32 + k] = (uint8_t)idx[r];
            gapT[r * 32 + k] = (uint32_t)(P[idx[r + 1]] - P[idx[r]]);
        }
    }
}

// ---------------------------------------------------------------- device pieces

// histogram of the lobe (w, M6) accumulators `lob` into H[0..124]; priv: 1000 words scratch
// not inlined: called at two sites (initial lobes, merged lobe), each call is thousands of
// instructions, so one copy of the code keeps the kernel's hot loops in the instruction cache
__device__ __noinline__ void hist_build(const long long* lob, const float* __restrict__ ux,
                                           const float* __restrict__ uy, const float* __restrict__ uz, int N,
                                           uint32_t* priv, uint16_t* H, int lane) {
    for (int w = lane; w < HB * 8; w += 32) priv[w] = 0u;
    const float wf = deq32(lob[0]);
    float S[6];
#pragma unroll
    for (int e = 0; e < 6; e++) S[e] = deq32(lob[1 + e]) / wf;
    const float L00 = sqrtf(pmax(S[0], 0.0f));
    const float L10 = L00 > 0.0f ? S[3] / L00 : 0.0f;
    const float L20 = L00 > 0.0f ? S[4] / L00 : 0.0f;
    const float L11 = sqrtf(pmax(S[1] - L10 * L10, 0.0f));
    const float L21 = L11 > 0.0f ? (S[5] - L20 * L10) / L11 : 0.0f;
    const float L22 = sqrtf(pmax((S[2] - L20 * L20) - L21 * L21, 0.0f));
    __syncwarp();
    uint8_t* pb = reinterpret_cast<uint8_t*>(priv);
    auto bin_uv = [&](float u0, float u1, float u2) {
        const float v0 = L00 * u0;
        const float v1 = L10 * u0 + L11 * u1;
        const float v2 = (L20 * u0 + L21 * u1) + L22 * u2;
        const float n2 = (v0 * v0 + v1 * v1) + v2 * v2;
        int b = 62;   // cell (2,2,2) when v = 0
        if (n2 > 0.0f) {
            b = hist_cell_fast(v0, v1, v2, n2);
            if (b < 0) b = hist_cell_pinned(v0, v1, v2, n2);   // rare: a component at a cell boundary
        }
        return b;
    };
    auto bin_of = [&](int s) { return bin_uv(ux[s], uy[s], uz[s]); };
    // four independent samples per step (ILP), the next step's table loads issued before this
    // step's arithmetic (software pipelining); the counter updates follow in sample order
    int s = lane;
    if (s + 96 < N) {
        float a[12];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            a[3 * q] = ux[s + 32 * q];
            a[3 * q + 1] = uy[s + 32 * q];
            a[3 * q + 2] = uz[s + 32 * q];
        }
        for (; s + 96 < N; s += 128) {
            float c[12];
#pragma unroll
            for (int q = 0; q < 12; q++) c[q] = a[q];
            if (s + 128 + 96 < N) {
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    a[3 * q] = ux[s + 128 + 32 * q];
                    a[3 * q + 1] = uy[s + 128 + 32 * q];
                    a[3 * q + 2] = uz[s + 128 + 32 * q];
                }
            }
            const int b0 = bin_uv(c[0], c[1], c[2]), b1 = bin_uv(c[3], c[4], c[5]);
            const int b2 = bin_uv(c[6], c[7], c[8]), b3 = bin_uv(c[9], c[10], c[11]);
            pb[b0 * 32 + lane] += 1;
            pb[b1 * 32 + lane] += 1;
            pb[b2 * 32 + lane] += 1;
            pb[b3 * 32 + lane] += 1;
        }
    }
    for (; s < N; s += 32) pb[bin_of(s) * 32 + lane] += 1;
    __syncwarp();
    for (int b = lane; b < HB; b += 32) {
        unsigned sum = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) sum = __dp4a(priv[b * 8 + q], 0x01010101u, sum);
        H[b] = (uint16_t)sum;
    }
    __syncwarp();
}

// d_hist(i, j_q) for up to 4 rows j_q at once (PREDICATES §10): lane k walks slice k, the
// table and H_i loads shared by the rows; exact 64-bit warp sums
template <int R>
__device__ __forceinline__ void hist_pairs(const uint16_t* Hi, const uint16_t* const (&Hj)[4],
                                           const uint32_t* __restrict__ pg, int lane,
                                           unsigned long long (&out)[4]) {
    int C[R];
    unsigned long long W[R];
#pragma unroll
    for (int q = 0; q < R; q++) {
        C[q] = 0;
        W[q] = 0;
    }
    static_assert(HR % 4 == 0, "slice steps in groups of four");
    for (int r0 = 0; r0 < HR; r0 += 4) {
        // four table words and their histogram reads issued before the dependent sums
        unsigned w[4];
        int hi[4], hj[4][R];
#pragma unroll
        for (int k = 0; k < 4; k++) w[k] = __ldg(pg + (r0 + k) * 32 + lane);   // (gap << 8) | cell
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int b = (int)(w[k] & 0xffu);
            hi[k] = Hi[b];
#pragma unroll
            for (int q = 0; q < R; q++) hj[k][q] = Hj[q][b];
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const unsigned g = w[k] >> 8;
#pragma unroll
            for (int q = 0; q < R; q++) {
                C[q] += hi[k] - hj[k][q];
                W[q] += (unsigned long long)(unsigned)(C[q] < 0 ? -C[q] : C[q]) * g;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < R; q++) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) W[q] += __shfl_xor_sync(0xffffffffu, W[q], o);
        out[q] = W[q];
    }
}

// distances of row i to the listed columns xs[0..m-1] (m <= 4), batched
// not inlined (two call sites, as hist_build)
__device__ __noinline__ void hist_row4(const uint16_t (*H)[128], int i, const int (&xs)[4], int m,
                                          const uint32_t* __restrict__ pg, int lane,
                                          unsigned long long (&out)[4]) {
    const uint16_t* Hj[4] = {H[xs[0]], H[xs[m > 1 ? 1 : 0]], H[xs[m > 2 ? 2 : 0]], H[xs[m > 3 ? 3 : 0]]};
    if (m == 4) hist_pairs<4>(H[i], Hj, pg, lane, out);
    else if (m == 3) hist_pairs<3>(H[i], Hj, pg, lane, out);
    else if (m == 2) hist_pairs<2>(H[i], Hj, pg, lane, out);
    else hist_pairs<1>(H[i], Hj, pg, lane, out);
}

// key = (d << 16) | (i << 8) | j orders by (d, i, j); d < 2^38 (32 slices x N x 2^20)
__device__ __forceinline__ unsigned long long hist_key(unsigned long long d, int i, int j) {
    return (d << 16) | (unsigned long long)((i << 8) | j);
}
constexpr unsigned long long HIST_RETIRED = 0xFFFFFFFFFFFFull << 16;

template <int K>
struct HistSmem {
    static constexpr int MAXN = 8 * K;
    static constexpr int MAXP = MAXN * (MAXN - 1) / 2;
    static constexpr int WARPS = K <= 4 ? 4 : 2;
    static constexpr size_t tables = 0;   // slice tables are read from global memory (L1)
    static constexpr size_t lob_bytes = MAXN * 7 * 8;
    static constexpr size_t H_bytes = MAXN * 128 * 2;
    static constexpr size_t priv_bytes = HB * 32;
    static constexpr size_t D_bytes = ((MAXP * 8 + 15) / 16) * 16;
    static constexpr size_t per_warp = lob_bytes + H_bytes + priv_bytes + D_bytes;
    static constexpr size_t total = tables + WARPS * per_warp;
};

template <int K>
__global__ void __launch_bounds__(128, 1)
k_sggxh_hist(const uint32_t* __restrict__ list, const unsigned* __restrict__ counts,
             const long long* __restrict__ cacc, const uint8_t* __restrict__ cncl,
             const long long* __restrict__ cclacc, int leaf, const uint32_t* __restrict__ start,
             uint8_t* __restrict__ pncl, long long* __restrict__ pclacc,
             const float* __restrict__ hu, int N, const uint32_t* __restrict__ gpg) {
    using SM = HistSmem<K>;
    constexpr int MAXN = SM::MAXN;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* base = smem_raw + SM::tables + wib * SM::per_warp;
    long long(*lob)[7] = reinterpret_cast<long long(*)[7]>(base);
    uint16_t(*H)[128] = reinterpret_cast<uint16_t(*)[128]>(base + SM::lob_bytes);
    uint32_t* priv = reinterpret_cast<uint32_t*>(base + SM::lob_bytes + SM::H_bytes);
    unsigned long long* D = reinterpret_cast<unsigned long long*>(base + SM::lob_bytes + SM::H_bytes + SM::priv_bytes);
    const float *ux = hu, *uy = hu + N, *uz = hu + 2 * N;
    const unsigned hi = counts[2];
    for (unsigned w = blockIdx.x * SM::WARPS + wib; w < hi; w += gridDim.x * SM::WARPS) {
        const uint64_t p = list[w];
        const uint32_t c0 = start[p], c1 = start[p + 1];
        int n = 0;
        // dendrogram leaves in child-slot order, w = 0 dropped (D17)
        if (leaf) {
            const int nch = (int)(c1 - c0);
            const bool has = lane < nch && cacc[7 * (uint64_t)(c0 + lane)] > 0;
            const unsigned bal = __ballot_sync(0xffffffffu, has);
            n = __popc(bal);
            if (has) {
                const int c = __popc(bal & ((1u << lane) - 1u));
#pragma unroll
                for (int e = 0; e < 7; e++) lob[c][e] = cacc[7 * (uint64_t)(c0 + lane) + e];
            }
        } else {
            const int slots = (int)(c1 - c0) * K;
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
                const unsigned bal = __ballot_sync(0xffffffffu, has);
                if (has) {
                    const int c = n + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
                    for (int e = 0; e < 7; e++) lob[c][e] = src[e];
                }
                n += __popc(bal);
            }
        }
        __syncwarp();
        for (int c = 0; c < n; c++) hist_build(lob[c], ux, uy, uz, N, priv, H[c], lane);
        // initial matrix: row i against columns j > i, four at a time
        for (int i = 0; i + 1 < n; i++)
            for (int j0 = i + 1; j0 < n; j0 += 4) {
                const int m = n - j0 < 4 ? n - j0 : 4;
                const int xs[4] = {j0, j0 + 1, j0 + 2, j0 + 3};
                unsigned long long d[4];
                hist_row4(H, i, xs, m, gpg, lane, d);
                if (lane < m) {
                    const int j = j0 + lane;
                    const unsigned long long dv = lane == 0 ? d[0] : lane == 1 ? d[1] : lane == 2 ? d[2] : d[3];
                    D[j * (j - 1) / 2 + i] = hist_key(dv, i, j);
                }
            }
        __syncwarp();
        const int np = n * (n - 1) / 2;
        unsigned long long alive = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
        for (int m = n; m > K; m--) {
            unsigned long long best = ~0ull;
            for (int t = lane; t < np; t += 32) {
                const unsigned long long key = D[t];
                best = key < best ? key : best;
            }
            const unsigned bh = (unsigned)(best >> 32);
            const unsigned dmin = __reduce_min_sync(0xffffffffu, bh);
            const unsigned lmin = __reduce_min_sync(0xffffffffu, bh == dmin ? (unsigned)best : 0xffffffffu);
            const int bi = (int)((lmin >> 8) & 0xff), bj = (int)(lmin & 0xff);
            if (lane < 7) lob[bi][lane] += lob[bj][lane];   // exact moment merge (D15)
            alive &= ~(1ull << bj);
            __syncwarp();
            if (m == K + 1) break;   // the last merge: no histogram or distance is read afterwards
            hist_build(lob[bi], ux, uy, uz, N, priv, H[bi], lane);   // fresh histogram of the merged S
            {   // new row d(bi, x) for the live x, four at a time
                unsigned long long rest = alive & ~(1ull << bi);
                while (rest) {
                    int xs[4] = {0, 0, 0, 0}, m = 0;
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (rest) {
                            xs[q] = __ffsll((long long)rest) - 1;
                            rest &= rest - 1;
                            m++;
                        }
                    unsigned long long d[4];
                    hist_row4(H, bi, xs, m, gpg, lane, d);
                    if (lane < m) {
                        const int x = lane == 0 ? xs[0] : lane == 1 ? xs[1] : lane == 2 ? xs[2] : xs[3];
                        const unsigned long long dv = lane == 0 ? d[0] : lane == 1 ? d[1] : lane == 2 ? d[2] : d[3];
                        const int a = x < bi ? x : bi, b2 = x < bi ? bi : x;
                        D[b2 * (b2 - 1) / 2 + a] = hist_key(dv, a, b2);
                    }
                }
            }
            for (int x = lane; x < n; x += 32)
                if (x != bj) {
                    const int a = x < bj ? x : bj, b2 = x < bj ? bj : x;
                    D[b2 * (b2 - 1) / 2 + a] = HIST_RETIRED | (unsigned long long)((a << 8) | b2);
                }
            __syncwarp();
        }
        int slot = 0;
        for (int cc = 0; cc < n; cc++) {
            if (!((alive >> cc) & 1ull)) continue;
            if (lane < 7) {
                const long long a = lob[cc][lane];
                pclacc[(p * K + slot) * 7 + lane] = a;
            }
            slot++;
        }
        if (lane == 0) pncl[p] = (uint8_t)slot;
        __syncwarp();
        (void)MAXN;
    }
}

template <int K>
static cudaError_t launch_hist_k(vox_ctx* c, const uint32_t* list, const unsigned* counts, const Level& C, int leaf,
                                 const uint32_t* start, Level& P) {
    using SM = HistSmem<K>;
    cudaError_t e = cudaFuncSetAttribute(k_sggxh_hist<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SM::total);
    if (e != cudaSuccess) return e;
    uint64_t nb = (P.n + SM::WARPS - 1) / SM::WARPS;
    nb = std::min<uint64_t>(std::max<uint64_t>(nb, 1), 148ull * 8);
    k_sggxh_hist<K><<<(unsigned)nb, SM::WARPS * 32, SM::total, c->stream>>>(
        list, counts, C.acc, C.ncl, C.clacc, leaf, start, P.ncl, P.clacc, c->d_hist_u, c->hist_n,
        c->d_hist_pg);
    return cudaGetLastError();
}

cudaError_t launch_sggxh_hist(vox_ctx* c, int K, const uint32_t* list, const unsigned* counts, const Level& C,
                              int leaf, const uint32_t* start, Level& P) {
    switch (K) {
        case 1: return launch_hist_k<1>(c, list, counts, C, leaf, start, P);
        case 2: return launch_hist_k<2>(c, list, counts, C, leaf, start, P);
        case 3: return launch_hist_k<3>(c, list, counts, C, leaf, start, P);
        case 4: return launch_hist_k<4>(c, list, counts, C, leaf, start, P);
        case 5: return launch_hist_k<5>(c, list, counts, C, leaf, start, P);
        case 6: return launch_hist_k<6>(c, list, counts, C, leaf, start, P);
        case 7: return launch_hist_k<7>(c, list, counts, C, leaf, start, P);
        default: return launch_hist_k<8>(c, list, counts, C, leaf, start, P);
    }
}

// Device tables are built once per (device, N) and kept for the process (like the event
// pool): creating a ctx in the histogram mode costs no host table work or copies after that.
struct HistTablesDev {
    float* u = nullptr;
    uint32_t* pg = nullptr;   // [124][32] (gap << 8) | cell
};
static std::mutex g_hist_mu;
static std::map<std::pair<int, int>, HistTablesDev> g_hist_tables;

cudaError_t upload_hist_tables(vox_ctx* c) {
    if (c->d_hist_u) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_hist_mu);
    HistTablesDev& T = g_hist_tables[{dev, c->hist_n}];
    if (!T.u) {
        std::vector<float> u;
        std::vector<uint8_t> perm;
        std::vector<uint32_t> gap;
        host_hist_tables(c->hist_n, u, perm, gap);
        std::vector<uint32_t> pg(perm.size());
        for (size_t x = 0; x < pg.size(); x++) pg[x] = (gap[x] << 8) | perm[x];   // gaps < 2^20
        HistTablesDev t;
        if ((e = cudaMalloc((void**)&t.u, u.size() * 4)) != cudaSuccess) return e;
        if ((e = cudaMalloc((void**)&t.pg, pg.size() * 4)) != cudaSuccess) return e;
        // synchronous copies from pageable host vectors (once per process, device and N)
        if ((e = cudaMemcpy(t.u, u.data(), u.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
        if ((e = cudaMemcpy(t.pg, pg.data(), pg.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
        T = t;
    }
    c->d_hist_u = T.u;
    c->d_hist_pg = T.pg;
    return cudaSuccess;
}

}  // namespace vox
