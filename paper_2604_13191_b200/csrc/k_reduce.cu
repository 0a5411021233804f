// k_reduce.cu -- gathering (§3.3 "ordered by second level block ID ... detect the
// vector positions where the ID changes"): the pairs of a call, appended per Morton bin by the
// emit kernels, are ranked within their bin and reduced into exact fixed-point accumulators
// (docs/PREDICATES.md §8) -- no global sort. Also merges a new leaf set into an existing one
// (D19) by a merge of the two sorted key arrays.
#include "vox_internal.cuh"

namespace vox {

VOX_DEBUG_TU(reduce)

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

// ---------------------------------------------------------------- merge of two leaf sets (D19)
// A (the existing leaves, n0) and B (the new call's, V) are sorted with unique keys. In the
// merged order (equal keys: A first), a_i sits at i + |{b < a_i}| and b_j at j + |{a < b_j}|;
// a key present in both becomes one voxel, so every position is shifted down by the number of
// such duplicate keys before it (an exclusive scan over A of dup_i). A duplicate b_j lands on
// its a_i's slot and adds its accumulators (exact integer sums).

// number of keys of k[0..n) below key (lower bound)
__device__ __forceinline__ uint64_t lower_bound(const uint64_t* __restrict__ k, uint64_t n, uint64_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (k[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_merge_rank(const uint64_t* __restrict__ ka, uint64_t n0, const uint64_t* __restrict__ kb,
                             uint64_t V, unsigned* __restrict__ dup, uint32_t* __restrict__ jb) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n0; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = lower_bound(kb, V, ka[i]);
        jb[i] = (uint32_t)j;
        dup[i] = (j < V && kb[j] == ka[i]) ? 1u : 0u;
    }
}

__global__ void k_merge_write_a(const uint64_t* __restrict__ ka, const long long* __restrict__ aa, uint64_t n0,
                                const uint32_t* __restrict__ jb, const unsigned* __restrict__ dscan,
                                uint64_t* __restrict__ okey, long long* __restrict__ oacc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n0; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t u = i + jb[i] - dscan[i];
        okey[u] = ka[i];
#pragma unroll
        for (int e = 0; e < 7; e++) oacc[7 * u + e] = aa[7 * i + e];
    }
}

__global__ void k_merge_write_b(const uint64_t* __restrict__ ka, uint64_t n0, const uint64_t* __restrict__ kb,
                                const long long* __restrict__ ba, uint64_t V, const unsigned* __restrict__ dscan,
                                uint64_t* __restrict__ okey, long long* __restrict__ oacc) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < V; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = lower_bound(ka, n0, kb[j]);
        const uint64_t u = j + i - dscan[i];
        if (i < n0 && ka[i] == kb[j]) {   // the key is in both sets: add into a_i's voxel
#pragma unroll
            for (int e = 0; e < 7; e++) oacc[7 * u + e] += ba[7 * j + e];
        } else {
            okey[u] = kb[j];
#pragma unroll
            for (int e = 0; e < 7; e++) oacc[7 * u + e] = ba[7 * j + e];
        }
    }
}

vox_status merge_into_leaf(vox_ctx* c, uint64_t* nkey, long long* nacc, uint64_t V) {
    Level& L0 = c->lv[0];
    if (V == 0) {
        dfree(c, nkey);
        dfree(c, nacc);
        return VOX_OK;
    }
    if (L0.n > 0) {
        // disjoint, ordered key ranges (the Morton parts of one call): concatenation
        uint64_t last = 0, first = 0;
        CK(readback(c, {{&last, L0.key + L0.n - 1, 8}, {&first, nkey, 8}}));
        if (first > last) {
            timer_begin(c, c->t_merge);
            const uint64_t tot = L0.n + V;
            Level M;
            M.n = tot;
            CK(dalloc(c, (void**)&M.key, tot * 8));
            CK(dalloc(c, (void**)&M.acc, tot * 56));
            CK(cudaMemcpyAsync(M.key, L0.key, L0.n * 8, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(M.key + L0.n, nkey, V * 8, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(M.acc, L0.acc, L0.n * 56, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(M.acc + 7 * L0.n, nacc, V * 56, cudaMemcpyDeviceToDevice, c->stream));
            dfree(c, nkey);
            dfree(c, nacc);
            free_level(c, L0);
            L0 = M;
            timer_end(c, c->t_merge);
            return VOX_OK;
        }
    }
    if (L0.n == 0) {
        free_level(c, L0);
        L0.n = V;
        L0.key = nkey;
        L0.acc = nacc;
        return VOX_OK;
    } else {
        timer_begin(c, c->t_merge);
        const uint64_t n0 = L0.n;
        unsigned* dup = nullptr;
        unsigned* dscan = nullptr;
        uint32_t* jb = nullptr;
        CK(dalloc(c, (void**)&dup, (n0 + 1) * 4));
        CK(dalloc(c, (void**)&dscan, (n0 + 1) * 4));
        CK(dalloc(c, (void**)&jb, n0 * 4));
        CK(cudaMemsetAsync(dup + n0, 0, 4, c->stream));
        k_merge_rank<<<grid_for(n0), 256, 0, c->stream>>>(L0.key, n0, nkey, V, dup, jb);
        CK(scan_excl_u32(c, dup, dscan, n0 + 1));
        unsigned D = 0;
        CK(readback(c, {{&D, dscan + n0, 4}}));
        const uint64_t VM = n0 + V - D;
        uint64_t* mkey = nullptr;
        long long* macc = nullptr;
        CK(dalloc(c, (void**)&mkey, VM * 8));
        CK(dalloc(c, (void**)&macc, VM * 56));
        k_merge_write_a<<<grid_for(n0), 256, 0, c->stream>>>(L0.key, L0.acc, n0, jb, dscan, mkey, macc);
        k_merge_write_b<<<grid_for(V), 256, 0, c->stream>>>(L0.key, n0, nkey, nacc, V, dscan, mkey, macc);
        c->st.launches += 3;
        CK(cudaGetLastError());
        dfree(c, dup);
        dfree(c, dscan);
        dfree(c, jb);
        dfree(c, nkey);
        dfree(c, nacc);
        free_level(c, L0);
        L0.n = VM;
        L0.key = mkey;
        L0.acc = macc;
        timer_end(c, c->t_merge);
    }
    return VOX_OK;
}

// ---------------------------------------------------------------- binned reduce
// Pairs were appended per bin (a Morton cell of 2^Lb voxels per edge, Lb <= 5, so a bin has at
// most 32768 voxels). Within a bin, the set of distinct keys is a bitmap over the bin's local
// Morton codes, and the position of a key in sorted order is the number of set bits below it
// (word prefix + popc), so the "sort" of P:242-248 becomes an O(1) rank per pair. Pass 1 counts
// distinct keys per bin; an exclusive scan gives every bin's first output slot; pass 2 sums the
// exact fixed-point contributions (§5, §7, §8) of each key in shared memory by rank and writes
// the bin's voxels contiguously in key order.

__global__ void k_group_sum(const unsigned long long* __restrict__ Wb, uint64_t nT, uint64_t group,
                            unsigned long long* __restrict__ WT) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nT; c += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long s = 0;
        for (uint64_t x = 0; x < group; x++) s += Wb[c * group + x];
        WT[c] = s;
    }
}


constexpr int BIN_THREADS = 128;

// Compact list of the non-empty bins (order irrelevant: every bin writes its own slots).
__global__ void k_bin_active(const unsigned* __restrict__ cnt, uint64_t nb, unsigned* __restrict__ list,
                             unsigned* __restrict__ nact) {
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb; b += (uint64_t)gridDim.x * blockDim.x) {
        const bool act = cnt[b] != 0;
        const unsigned m = __ballot_sync(__activemask(), act);
        if (!m) continue;
        const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(nact, (unsigned)__popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (act) list[base + __popc(m & ((1u << lane) - 1u))] = (unsigned)b;
    }
}

// pass 1: distinct keys per bin (bitmap popcount); also totals the pairs
__global__ void __launch_bounds__(BIN_THREADS)
k_bin_count(const uint64_t* __restrict__ keys, const unsigned long long* __restrict__ off,
            const unsigned* __restrict__ cnt, const unsigned* __restrict__ alist, const unsigned* __restrict__ nact,
            int lbits, unsigned* __restrict__ vcount, unsigned long long* __restrict__ npairs) {
    extern __shared__ unsigned s_bm[];
    __shared__ unsigned s_red[BIN_THREADS / 32];
    const int words = lbits >= 5 ? (1 << (lbits - 5)) : 1;
    const uint64_t lmask = (1ull << lbits) - 1ull;
    const unsigned na = *nact;
    for (unsigned ai = blockIdx.x; ai < na; ai += gridDim.x) {
        const unsigned b = alist[ai];
        const unsigned n = cnt[b];
        for (int w = threadIdx.x; w < words; w += blockDim.x) s_bm[w] = 0u;
        __syncthreads();
        const uint64_t o = off[b];
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned lk = (unsigned)(keys[o + i] & lmask);
            atomicOr(&s_bm[lk >> 5], 1u << (lk & 31));
        }
        __syncthreads();
        unsigned c = 0;
        for (int w = threadIdx.x; w < words; w += blockDim.x) c += __popc(s_bm[w]);
        c = __reduce_add_sync(0xffffffffu, c);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned t = 0;
            for (int q = 0; q < BIN_THREADS / 32; q++) t += s_red[q];
            vcount[b] = t;
            atomicAdd(npairs, (unsigned long long)n);
        }
        __syncthreads();
    }
}

constexpr int BIN_NMAX = 6144;    // pairs of a bin handled by the in-shared-memory counting sort
constexpr int BIN_VMAX = 4096;    // distinct keys of such a bin (a 16^3 bin has at most 4096)
constexpr int BIN_CHUNK = 384;    // voxels per pass of the fallback path (bins with more pairs)
constexpr int BIN_WORDS = 1024;   // bitmap words reserved (32^3 bins)

// exclusive prefix of popcounts of the bitmap words (block scan over <= 1024 words)
__device__ __forceinline__ void bitmap_prefix(const unsigned* bm, unsigned* wpre, int words, unsigned* s_wsum) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int per = (words + BIN_THREADS - 1) / BIN_THREADS;
    const int w0 = threadIdx.x * per;
    unsigned loc = 0;
    for (int q = 0; q < per; q++)
        if (w0 + q < words) loc += __popc(bm[w0 + q]);
    unsigned inc = loc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) s_wsum[wid] = inc;
    __syncthreads();
    unsigned run = inc - loc;
    for (int q = 0; q < wid; q++) run += s_wsum[q];
    for (int q = 0; q < per; q++)
        if (w0 + q < words) {
            wpre[w0 + q] = run;
            run += __popc(bm[w0 + q]);
        }
    __syncthreads();
}

template <class W>
__device__ __forceinline__ unsigned key_rank(const unsigned* bm, const W* wpre, unsigned lk) {
    const unsigned w = lk >> 5, bit = lk & 31;
    return wpre[w] + __popc(bm[w] & ((1u << bit) - 1u));
}

// one voxel's exact sums over its pairs (§5, §7, §8), written as a key-ordered output row
// (the fp32 views are produced on demand from the accumulators, launch_finalize)
__device__ __forceinline__ void emit_voxel(uint64_t key, const long long (&a)[7], uint64_t r, uint64_t* okey,
                                          long long* oacc) {
    okey[r] = key;
#pragma unroll
    for (int e = 0; e < 7; e++) oacc[7 * r + e] = a[e];
}

__device__ __forceinline__ void add_pair(uint64_t val, const float4* __restrict__ ptab, long long (&a)[7]) {
    const float4 pt = ptab[(uint32_t)val];
    const float wgt = __uint_as_float((uint32_t)(val >> 32));
    const float mass = pt.w * wgt;
    const float mx = mass * pt.x, my = mass * pt.y, mz = mass * pt.z;
    a[0] += q32(mass);
    a[1] += q32(mx * pt.x);
    a[2] += q32(my * pt.y);
    a[3] += q32(mz * pt.z);
    a[4] += q32(mx * pt.y);
    a[5] += q32(mx * pt.z);
    a[6] += q32(my * pt.z);
}

// pass 2: per bin, ranks from the bitmap; bins of <= BIN_NMAX pairs and <= BIN_VMAX keys are
// counting-sorted by rank in shared memory and each thread then sums whole voxels in
// registers (no 64-bit atomics); larger bins take the chunked path with shared atomics.
__global__ void __launch_bounds__(BIN_THREADS)
k_bin_reduce(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, const float4* __restrict__ ptab,
             const unsigned long long* __restrict__ off, const unsigned* __restrict__ cnt,
             const unsigned* __restrict__ alist, const unsigned* __restrict__ nact,
             const unsigned* __restrict__ voff, int lbits, uint64_t* __restrict__ okey,
             long long* __restrict__ oacc) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int words = lbits >= 5 ? (1 << (lbits - 5)) : 1;
    unsigned* bm = reinterpret_cast<unsigned*>(s_raw);                      // [words]
    unsigned* wpre = bm + words;                                            // [words]
    unsigned* cur = wpre + words;                                           // [BIN_VMAX + 1]
    unsigned short* sidx = reinterpret_cast<unsigned short*>(cur + BIN_VMAX + 1);   // [BIN_NMAX]
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(cur);   // fallback: [BIN_CHUNK][7]
    unsigned short* lkey = reinterpret_cast<unsigned short*>(acc + BIN_CHUNK * 7);   // fallback: [BIN_CHUNK]
    __shared__ unsigned s_wsum[BIN_THREADS / 32];
    const uint64_t lmask = (1ull << lbits) - 1ull;
    const unsigned na = *nact;
    for (unsigned ai = blockIdx.x; ai < na; ai += gridDim.x) {
        const unsigned b = alist[ai];
        const unsigned n = cnt[b];
        const uint64_t o = off[b];
        const unsigned vb = voff[b], V = voff[b + 1] - vb;
        const uint64_t kbase = (uint64_t)b << lbits;
        for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0u;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned lk = (unsigned)(keys[o + i] & lmask);
            atomicOr(&bm[lk >> 5], 1u << (lk & 31));
        }
        __syncthreads();
        bitmap_prefix(bm, wpre, words, s_wsum);
        if (n <= BIN_NMAX && V <= BIN_VMAX) {
            for (unsigned r = threadIdx.x; r <= V; r += blockDim.x) cur[r] = 0u;
            __syncthreads();
            for (unsigned i = threadIdx.x; i < n; i += blockDim.x)
                atomicAdd(&cur[key_rank(bm, wpre, (unsigned)(keys[o + i] & lmask)) + 1], 1u);
            __syncthreads();
            // inclusive scan of cur[1..V] -> cur[r] = first slot of rank r (cur[0] = 0)
            {
                const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
                const unsigned per = (V + 1 + BIN_THREADS - 1) / BIN_THREADS;
                const unsigned r0 = threadIdx.x * per;
                unsigned loc = 0;
                for (unsigned q = 0; q < per; q++)
                    if (r0 + q <= V) loc += cur[r0 + q];
                unsigned inc = loc;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += y;
                }
                if (lane == 31) s_wsum[wid] = inc;
                __syncthreads();
                unsigned run = inc - loc;
                for (int q = 0; q < wid; q++) run += s_wsum[q];
                for (unsigned q = 0; q < per; q++)
                    if (r0 + q <= V) {
                        run += cur[r0 + q];
                        cur[r0 + q] = run;
                    }
                __syncthreads();
            }
            // scatter pair indices by rank; afterwards cur[r] = end of rank r's run
            for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
                const unsigned r = key_rank(bm, wpre, (unsigned)(keys[o + i] & lmask));
                VOX_DCHECK(r < V, 1);
                const unsigned slot = atomicAdd(&cur[r], 1u);
                VOX_DCHECK(slot < n && slot < BIN_NMAX, 2);
                sidx[slot] = (unsigned short)i;
            }
            __syncthreads();
            for (unsigned r = threadIdx.x; r < V; r += blockDim.x) {
                const unsigned p0 = r == 0 ? 0u : cur[r - 1], p1 = cur[r];
                long long a[7] = {0, 0, 0, 0, 0, 0, 0};
                for (unsigned p = p0; p < p1; p++) add_pair(vals[o + sidx[p]], ptab, a);
                emit_voxel(keys[o + sidx[p0]], a, (uint64_t)vb + r, okey, oacc);
            }
            __syncthreads();
        } else {
            for (unsigned r0 = 0; r0 < V; r0 += BIN_CHUNK) {
                const unsigned rn = V - r0 < BIN_CHUNK ? V - r0 : BIN_CHUNK;
                for (unsigned x = threadIdx.x; x < rn * 7; x += blockDim.x) acc[x] = 0ull;
                for (int w = threadIdx.x; w < words; w += blockDim.x) {
                    unsigned m = bm[w];
                    unsigned r = wpre[w];
                    while (m) {
                        const int bit = __ffs(m) - 1;
                        m &= m - 1;
                        if (r >= r0 && r < r0 + rn) lkey[r - r0] = (unsigned short)((w << 5) | bit);
                        r++;
                    }
                }
                __syncthreads();
                for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
                    const unsigned r = key_rank(bm, wpre, (unsigned)(keys[o + i] & lmask));
                    if (r < r0 || r >= r0 + rn) continue;
                    long long a[7] = {0, 0, 0, 0, 0, 0, 0};
                    add_pair(vals[o + i], ptab, a);
                    unsigned long long* d = acc + 7 * (r - r0);
#pragma unroll
                    for (int e = 0; e < 7; e++) atomicAdd(d + e, (unsigned long long)a[e]);
                }
                __syncthreads();
                for (unsigned x = threadIdx.x; x < rn; x += blockDim.x) {
                    long long a[7];
#pragma unroll
                    for (int e = 0; e < 7; e++) a[e] = (long long)acc[7 * x + e];
                    emit_voxel(kbase | lkey[x], a, (uint64_t)vb + r0 + x, okey, oacc);
                }
                __syncthreads();
            }
        }
    }
}

// Warp-per-bin variant for the common small bins (no block barriers): each warp owns a bin
// of <= WB_NMAX pairs and <= WB_VMAX distinct keys with a private bitmap / rank table in
// shared memory. Bins above the limits are listed for k_bin_reduce (block per bin).
constexpr int WB_WARPS = 4;
constexpr int WB_NMAX = 1536;
constexpr int WB_VMAX = 1024;

__global__ void __launch_bounds__(WB_WARPS * 32)
k_bin_reduce_warp(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals,
                  const float4* __restrict__ ptab, const unsigned long long* __restrict__ off,
                  const unsigned* __restrict__ cnt, const unsigned* __restrict__ alist,
                  const unsigned* __restrict__ nact, const unsigned* __restrict__ voff, int lbits,
                  unsigned* __restrict__ big, unsigned* __restrict__ nbig, uint64_t* __restrict__ okey,
                  long long* __restrict__ oacc) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int words = lbits >= 5 ? (1 << (lbits - 5)) : 1;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // word prefixes as u16 (a warp bin has <= WB_VMAX keys): 2 B per bitmap word
    const size_t per_warp = ((size_t)words * 6 + (WB_VMAX + 1) * 4 + WB_NMAX * 2 + 15) & ~(size_t)15;
    unsigned* bm = reinterpret_cast<unsigned*>(s_raw + wib * per_warp);
    unsigned* cur = bm + words;
    uint16_t* wpre = reinterpret_cast<uint16_t*>(cur + WB_VMAX + 1);
    unsigned short* sidx = reinterpret_cast<unsigned short*>(wpre + words);
    const uint64_t lmask = (1ull << lbits) - 1ull;
    const unsigned na = *nact;
    for (unsigned ai = blockIdx.x * WB_WARPS + wib; ai < na; ai += gridDim.x * WB_WARPS) {
        const unsigned b = alist[ai];
        const unsigned n = cnt[b];
        const unsigned vb = voff[b], V = voff[b + 1] - vb;
        if (n > WB_NMAX || V > WB_VMAX) {
            if (lane == 0) big[atomicAdd(nbig, 1u)] = b;
            continue;
        }
        const uint64_t o = off[b];
        for (int w = lane; w < words; w += 32) bm[w] = 0u;
        for (unsigned r = lane; r <= V; r += 32) cur[r] = 0u;
        __syncwarp();
        for (unsigned i = lane; i < n; i += 32) {
            const unsigned lk = (unsigned)(keys[o + i] & lmask);
            atomicOr(&bm[lk >> 5], 1u << (lk & 31));
        }
        __syncwarp();
        {   // exclusive popcount prefix over the words: contiguous chunk per lane + warp scan
            const int per = (words + 31) / 32, w0 = lane * per;
            unsigned loc = 0;
            for (int q = 0; q < per; q++)
                if (w0 + q < words) loc += __popc(bm[w0 + q]);
            unsigned inc = loc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += y;
            }
            unsigned run = inc - loc;
            for (int q = 0; q < per; q++)
                if (w0 + q < words) {
                    wpre[w0 + q] = (uint16_t)run;
                    run += __popc(bm[w0 + q]);
                }
        }
        __syncwarp();
        for (unsigned i = lane; i < n; i += 32)
            atomicAdd(&cur[key_rank(bm, wpre, (unsigned)(keys[o + i] & lmask)) + 1], 1u);
        __syncwarp();
        {   // inclusive scan of cur[0..V] -> cur[r] = first slot of rank r
            const unsigned per = (V + 1 + 31) / 32, r0 = lane * per;
            unsigned loc = 0;
            for (unsigned q = 0; q < per; q++)
                if (r0 + q <= V) loc += cur[r0 + q];
            unsigned inc = loc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += y;
            }
            unsigned run = inc - loc;
            for (unsigned q = 0; q < per; q++)
                if (r0 + q <= V) {
                    run += cur[r0 + q];
                    cur[r0 + q] = run;
                }
        }
        __syncwarp();
        for (unsigned i = lane; i < n; i += 32) {
            const unsigned r = key_rank(bm, wpre, (unsigned)(keys[o + i] & lmask));
            VOX_DCHECK(r < V, 1);
            const unsigned slot = atomicAdd(&cur[r], 1u);
            VOX_DCHECK(slot < n && slot < WB_NMAX, 2);
            sidx[slot] = (unsigned short)i;
        }
        __syncwarp();
        for (unsigned r = lane; r < V; r += 32) {
            const unsigned p0 = r == 0 ? 0u : cur[r - 1], p1 = cur[r];
            long long a[7] = {0, 0, 0, 0, 0, 0, 0};
            for (unsigned p = p0; p < p1; p++) add_pair(vals[o + sidx[p]], ptab, a);
            emit_voxel(keys[o + sidx[p0]], a, (uint64_t)vb + r, okey, oacc);
        }
        __syncwarp();
    }
}

// Top-cell candidate counts (sum of the bins of each top cell) for the shard plan.
vox_status bin_topcells(vox_ctx* c, const unsigned long long* Wb, int Lb, std::vector<uint64_t>& WT) {
    const uint64_t nT = 1ull << (3 * c->T);
    const uint64_t group = 1ull << (3 * (c->g.logN - Lb - c->T));
    unsigned long long* dWT = nullptr;
    CK(dalloc(c, (void**)&dWT, nT * 8));
    k_group_sum<<<grid_for(nT), 256, 0, c->stream>>>(Wb, nT, group, dWT);
    c->st.launches++;
    WT.resize(nT);
    CK(cudaMemcpyAsync(WT.data(), dWT, nT * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(ssync(c));
    dfree(c, dWT);
    return VOX_OK;
}

// Capacity offsets of the bins of this rank's top cells; *cap_out = total (one 8-byte read).
vox_status bin_offsets(vox_ctx* c, const unsigned long long* Wb, int Lb, unsigned long long** off_out,
                       uint64_t* cap_out) {
    const uint64_t nb = 1ull << (3 * (c->g.logN - Lb));
    const int gshift = 3 * (c->g.logN - Lb - c->T);
    unsigned long long* off = nullptr;
    CK(dalloc(c, (void**)&off, (nb + 1) * 8));
    CK(scan_bin_caps(c, Wb, nb, gshift, c->cell_lo, c->cell_hi, off));   // caps of the rank's cells, scanned
    unsigned long long cap = 0;
    CK(readback(c, {{&cap, off + nb, 8}}));
    *off_out = off;
    *cap_out = cap;
    return VOX_OK;
}

vox_status reduce_bins(vox_ctx* c, const uint64_t* keys, const uint64_t* vals, Bins bins, uint64_t nb,
                       const float4* ptab, LeafSet& out) {
    const int lbits = bins.shift;
    const int words = lbits >= 5 ? (1 << (lbits - 5)) : 1;
    unsigned* vcount = nullptr;
    unsigned* voff = nullptr;
    unsigned long long* npairs = nullptr;
    timer_begin(c, c->t_sort);
    CK(dalloc(c, (void**)&vcount, (nb + 1) * 4));
    CK(dalloc(c, (void**)&voff, (nb + 1) * 4));
    CK(dalloc(c, (void**)&npairs, 16));
    unsigned* alist = nullptr;
    CK(dalloc(c, (void**)&alist, nb * 4));
    unsigned* nact = reinterpret_cast<unsigned*>(npairs + 1);
    CK(cudaMemsetAsync(npairs, 0, 16, c->stream));
    CK(cudaMemsetAsync(vcount, 0, (nb + 1) * 4, c->stream));
    k_bin_active<<<grid_for(nb), 256, 0, c->stream>>>(bins.cnt, nb, alist, nact);
    const unsigned grid = (unsigned)std::min<uint64_t>(nb, 148ull * 16);
    k_bin_count<<<grid, BIN_THREADS, words * 4, c->stream>>>(keys, bins.off, bins.cnt, alist, nact, lbits, vcount,
                                                             npairs);
    CK(scan_excl_u32(c, vcount, voff, nb + 1));
    c->st.launches += 2;
    unsigned V = 0;
    unsigned long long P = 0;
    CK(readback(c, {{&V, voff + nb, 4}, {&P, npairs, 8}}));
    timer_end(c, c->t_sort);
    c->st.pairs += P;
    timer_begin(c, c->t_reduce);
    uint64_t* nkey = nullptr;
    long long* nacc = nullptr;
    CK(dalloc(c, (void**)&nkey, (uint64_t)V * 8));
    CK(dalloc(c, (void**)&nacc, (uint64_t)V * 56));
    // small bins: warp per bin; the others (listed by it) then get a block each
    unsigned* big = nullptr;
    CK(dalloc(c, (void**)&big, nb * 4 + 4));
    unsigned* nbig = big + nb;
    CK(cudaMemsetAsync(nbig, 0, 4, c->stream));
    const size_t wsm = (size_t)WB_WARPS * (((size_t)words * 6 + (WB_VMAX + 1) * 4 + WB_NMAX * 2 + 15) & ~(size_t)15);
    CK(cudaFuncSetAttribute(k_bin_reduce_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
    const unsigned wgrid = (unsigned)std::min<uint64_t>((nb + WB_WARPS - 1) / WB_WARPS, 148ull * 32);
    k_bin_reduce_warp<<<wgrid, WB_WARPS * 32, wsm, c->stream>>>(keys, vals, ptab, bins.off, bins.cnt, alist, nact,
                                                                voff, lbits, big, nbig, nkey, nacc);
    const size_t smem = 2 * (size_t)words * 4 + (BIN_VMAX + 1) * 4 + BIN_NMAX * 2 + 16;
    static_assert(BIN_CHUNK * 7 * 8 + BIN_CHUNK * 2 <= (BIN_VMAX + 1) * 4 + BIN_NMAX * 2, "fallback must fit");
    CK(cudaFuncSetAttribute(k_bin_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_bin_reduce<<<grid, BIN_THREADS, smem, c->stream>>>(keys, vals, ptab, bins.off, bins.cnt, big, nbig, voff,
                                                         lbits, nkey, nacc);
    c->st.launches += 2;
    CK(cudaGetLastError());
    timer_end(c, c->t_reduce);
    dfree(c, vcount);
    dfree(c, voff);
    dfree(c, npairs);
    dfree(c, alist);
    dfree(c, big);
    out.key = nkey;
    out.acc = nacc;
    out.n = V;
    return VOX_OK;
}

}  // namespace vox
