// k_scan.cu -- exclusive prefix sums for the per-call offsets of the path: pair-bin capacity
// offsets, per-bin voxel offsets, triangle candidate offsets, and the run heads of a sorted
// key array (the parents of a pyramid level: "parent = key >> 3" runs over the
// Morton-sorted children). Hand-written so that no library kernel runs on the per-call path.
//
// Reduce-then-scan over warp chunks of 32 x SCAN_ROWS consecutive elements, read row by row
// (each row a coalesced 32-element load): (1) every chunk sums its values, (2) the chunk sums
// are scanned (one block, or recursively the same way when there are many), (3) every chunk
// recomputes its values and emits each with its exclusive prefix: warp inclusive scan of the
// row plus the running carry. Values come from a functor (they can be computed on the fly,
// e.g. run-head flags from keys), so no input array is needed; all sums are exact integer
// sums. (Measured alternatives, not kept: a single-pass decoupled look-back was 2-4x slower at
// these sizes, bound by its look-back chain; thread-contiguous 16-element tiles missed L1.)
#include "vox_internal.cuh"

namespace vox {

constexpr int SCAN_WARPS = 8;
constexpr int SCAN_ROWS = 32;
constexpr uint64_t SCAN_CHUNK = 32ull * SCAN_ROWS;   // elements per warp chunk

// F: __device__ uint64_t value(uint64_t i) const;  void output(uint64_t i, uint64_t excl, uint64_t v) const
template <class F>
__global__ void __launch_bounds__(SCAN_WARPS * 32) k_scan_reduce(F f, uint64_t n, unsigned long long* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const uint64_t ch = blockIdx.x * (uint64_t)SCAN_WARPS + (threadIdx.x >> 5);
    const uint64_t base = ch * SCAN_CHUNK;
    if (base >= n) return;
    unsigned long long t = 0;
#pragma unroll 4
    for (int r = 0; r < SCAN_ROWS; r++) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        if (i < n) t += f.value(i);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) part[ch] = t;
}

// exclusive scan of up to SCAN_SMALL chunk sums in one block (in place); thread t owns a
// contiguous run of them
constexpr uint64_t SCAN_SMALL = 1024ull * 16;
__global__ void __launch_bounds__(1024) k_scan_parts(unsigned long long* __restrict__ part, uint64_t m) {
    __shared__ unsigned long long s_warp[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t per = (m + 1023) / 1024, t0 = threadIdx.x * per;
    unsigned long long t = 0;
    for (uint64_t q = 0; q < per; q++)
        if (t0 + q < m) t += part[t0 + q];
    unsigned long long incl = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    unsigned long long run = incl - t;
    for (int w = 0; w < wid; w++) run += s_warp[w];
    for (uint64_t q = 0; q < per; q++)
        if (t0 + q < m) {
            const unsigned long long v = part[t0 + q];
            part[t0 + q] = run;
            run += v;
        }
}

template <class F>
__global__ void __launch_bounds__(SCAN_WARPS * 32)
k_scan_apply(F f, uint64_t n, const unsigned long long* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const uint64_t ch = blockIdx.x * (uint64_t)SCAN_WARPS + (threadIdx.x >> 5);
    const uint64_t base = ch * SCAN_CHUNK;
    if (base >= n) return;
    unsigned long long carry = part[ch];
    for (int r = 0; r < SCAN_ROWS; r++) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        if (base + (uint64_t)r * 32 >= n) break;
        const unsigned long long v = i < n ? f.value(i) : 0ull;
        unsigned long long incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        if (i < n) f.output(i, carry + incl - v, v);
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

template <class F>
static cudaError_t run_scan(vox_ctx* c, const F& f, uint64_t n);

// exclusive scan of an array of chunk sums in place (recursive for many chunks)
struct InPlaceU64 {
    unsigned long long* a;
    unsigned long long* out;
    __device__ uint64_t value(uint64_t i) const { return a[i]; }
    __device__ void output(uint64_t i, uint64_t excl, uint64_t) const { out[i] = excl; }
};
static cudaError_t scan_parts(vox_ctx* c, unsigned long long* part, uint64_t m) {
    if (m <= SCAN_SMALL) {
        k_scan_parts<<<1, 1024, 0, c->stream>>>(part, m);
        c->st.launches++;
        return cudaGetLastError();
    }
    unsigned long long* tmp = nullptr;
    cudaError_t e = dalloc(c, (void**)&tmp, m * 8);
    if (e != cudaSuccess) return e;
    if ((e = run_scan(c, InPlaceU64{part, tmp}, m)) != cudaSuccess) return e;
    e = cudaMemcpyAsync(part, tmp, m * 8, cudaMemcpyDeviceToDevice, c->stream);
    dfree(c, tmp);
    return e;
}

template <class F>
static cudaError_t run_scan(vox_ctx* c, const F& f, uint64_t n) {
    if (n == 0) return cudaSuccess;
    const uint64_t chunks = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
    const unsigned blocks = (unsigned)((chunks + SCAN_WARPS - 1) / SCAN_WARPS);
    unsigned long long* part = nullptr;
    cudaError_t e = dalloc(c, (void**)&part, chunks * 8);
    if (e != cudaSuccess) return e;
    k_scan_reduce<F><<<blocks, SCAN_WARPS * 32, 0, c->stream>>>(f, n, part);
    c->st.launches++;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = scan_parts(c, part, chunks)) != cudaSuccess) return e;
    k_scan_apply<F><<<blocks, SCAN_WARPS * 32, 0, c->stream>>>(f, n, part);
    c->st.launches++;
    e = cudaGetLastError();
    dfree(c, part);
    return e;
}

// ---- exclusive sum of a u64 array (in[n - 1] is usually a 0 pad so that out[n - 1] = total)
struct ExclU64 {
    const unsigned long long* in;
    unsigned long long* out;
    __device__ uint64_t value(uint64_t i) const { return in[i]; }
    __device__ void output(uint64_t i, uint64_t excl, uint64_t) const { out[i] = excl; }
};
cudaError_t scan_excl_u64(vox_ctx* c, const unsigned long long* in, unsigned long long* out, uint64_t n) {
    return run_scan(c, ExclU64{in, out}, n);
}

// ---- exclusive sum of a u32 array
struct ExclU32 {
    const unsigned* in;
    unsigned* out;
    __device__ uint64_t value(uint64_t i) const { return in[i]; }
    __device__ void output(uint64_t i, uint64_t excl, uint64_t) const { out[i] = (unsigned)excl; }
};
cudaError_t scan_excl_u32(vox_ctx* c, const unsigned* in, unsigned* out, uint64_t n) {
    return run_scan(c, ExclU32{in, out}, n);
}

// ---- capacity offsets of the pair bins of this rank's top cells: value = the bin's exact
// candidate count if its top cell (b >> gshift) is in [lo, hi), else 0; out[nb] = total
struct BinCaps {
    const unsigned long long* Wb;
    unsigned long long* off;
    uint64_t nb, lo, hi;
    int gshift;
    __device__ uint64_t value(uint64_t b) const {
        const uint64_t top = b >> gshift;
        return (b < nb && top >= lo && top < hi) ? Wb[b] : 0ull;
    }
    __device__ void output(uint64_t b, uint64_t excl, uint64_t) const { off[b] = excl; }
};
cudaError_t scan_bin_caps(vox_ctx* c, const unsigned long long* Wb, uint64_t nb, int gshift, uint64_t lo, uint64_t hi,
                          unsigned long long* off) {
    return run_scan(c, BinCaps{Wb, off, nb, lo, hi, gshift}, nb + 1);
}

// ---- run heads of a sorted key array: a head is the first child of each parent (key >> 3);
// the h-th head writes start[h] = its index and pkey[h] = its parent key; the last element
// closes start[V] = n and writes the parent count V
struct RunHeads {
    const uint64_t* key;
    uint32_t* start;
    uint64_t* pkey;
    uint32_t* total;
    uint64_t n;
    __device__ uint64_t value(uint64_t i) const {
        return (i == 0 || (key[i] >> 3) != (key[i - 1] >> 3)) ? 1ull : 0ull;
    }
    __device__ void output(uint64_t i, uint64_t excl, uint64_t v) const {
        if (v) {
            start[excl] = (uint32_t)i;
            pkey[excl] = key[i] >> 3;
        }
        if (i == n - 1) {
            start[excl + v] = (uint32_t)n;
            *total = (uint32_t)(excl + v);
        }
    }
};
cudaError_t scan_run_heads(vox_ctx* c, const uint64_t* key, uint64_t n, uint32_t* start, uint64_t* pkey,
                           uint32_t* total) {
    return run_scan(c, RunHeads{key, start, pkey, total, n}, n);
}

}  // namespace vox
