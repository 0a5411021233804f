// vox_internal.cuh -- internal declarations of libvox (product path; shares nothing with oracle/).
//
// All floating-point code in this library is compiled with -fmad=false, -prec-div=true,
// -prec-sqrt=true and without fast-math, so every expression below is the pinned
// sequence of IEEE binary32 operations of docs/PREDICATES.md.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <initializer_list>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/vox.h"

#define VOX_MAX_LEVELS 14
#define VOX_MAX_K 8
#define VOX_SLICES 32

// device error flags (bitmask)
#define VOX_EFLAG_NONFINITE 1u
#define VOX_EFLAG_NEG_RADIUS 2u
#define VOX_EFLAG_TOO_MANY_CAND 4u
#define VOX_EFLAG_ZERO_DIR 8u
#define VOX_EFLAG_OVERFLOW 16u

namespace vox {

// NVTX range for the lifetime of a scope (one per C-ABI call and per pyramid level), so an
// nsys / ncu timeline shows the library's calls; a no-op unless a tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define VOX_RANGE(name) ::vox::NvtxRange vox_nvtx_range_(name)

// Bounds checks of a debug build (-DVOX_DEBUG, e.g. VOX_NVCC_EXTRA=-DVOX_DEBUG): a failed check
// sets bit `bit` of a per-translation-unit device word; vox_debug_flags ORs them (compute-
// sanitizer is closed on the GPU pool, so the library checks its own shared-memory and slot
// indices). Release builds compile the checks out.
#ifdef VOX_DEBUG
#define VOX_DEBUG_TU(name)                                                          \
    static __device__ unsigned g_vox_dbg;                                           \
    unsigned debug_read_##name() {                                                  \
        unsigned v = 0;                                                             \
        cudaMemcpyFromSymbol(&v, g_vox_dbg, 4);                                     \
        const unsigned z = 0;                                                       \
        cudaMemcpyToSymbol(g_vox_dbg, &z, 4);                                       \
        return v;                                                                   \
    }
#define VOX_DCHECK(cond, bit)                                      \
    do {                                                           \
        if (!(cond)) atomicOr(&g_vox_dbg, 1u << (bit));            \
    } while (0)
#else
#define VOX_DEBUG_TU(name) \
    unsigned debug_read_##name() { return 0; }
#define VOX_DCHECK(cond, bit) \
    do {                      \
    } while (0)
#endif
unsigned debug_read_fiber();
unsigned debug_read_reduce();
unsigned debug_read_lod();

// ---------------------------------------------------------------- pinned helpers (PREDICATES)

__host__ __device__ __forceinline__ float pmin(float a, float b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ float pmax(float a, float b) { return a > b ? a : b; }

// §8 fixed point: q(x) = round-to-nearest-even(x * 2^32)
__device__ __forceinline__ long long q32(float x) { return __float2ll_rn(x * 4294967296.0f); }
__device__ __forceinline__ float deq32(long long a) { return __ll2float_rn(a) * 2.3283064365386963e-10f; }

// §2 Morton encoding (x in bit 0) by bit spreading
__host__ __device__ __forceinline__ uint64_t spread3(uint32_t v) {
    uint64_t x = v & 0x1fffffu;
    x = (x | (x << 32)) & 0x1f00000000ffffull;
    x = (x | (x << 16)) & 0x1f0000ff0000ffull;
    x = (x | (x << 8)) & 0x100f00f00f00f00full;
    x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}
__host__ __device__ __forceinline__ uint64_t morton3(uint32_t i, uint32_t j, uint32_t k) {
    return spread3(i) | (spread3(j) << 1) | (spread3(k) << 2);
}
// §2 Morton key from a shared 256-entry table of 8-bit bit spreads (coordinates < 2^16: two
// lookups per axis) -- the same bits as morton3 with a quarter of its 64-bit shift/mask steps.
// mtab_init fills the table (whole block, then a barrier: call it before any divergence).
__device__ __forceinline__ uint64_t morton3_tab(const uint64_t* __restrict__ tab, uint32_t i, uint32_t j, uint32_t k) {
    const uint64_t x = tab[i & 255u] | (tab[(i >> 8) & 255u] << 24);
    const uint64_t y = tab[j & 255u] | (tab[(j >> 8) & 255u] << 24);
    const uint64_t z = tab[k & 255u] | (tab[(k >> 8) & 255u] << 24);
    return x | (y << 1) | (z << 2);
}
__device__ __forceinline__ void mtab_init(uint64_t* tab) {
    for (int t = threadIdx.x; t < 256; t += blockDim.x) tab[t] = spread3((uint32_t)t);
    __syncthreads();
}
__host__ __device__ __forceinline__ uint32_t compact3(uint64_t x) {
    x &= 0x1249249249249249ull;
    x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
    x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
    x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
    x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
    x = (x ^ (x >> 32)) & 0x1fffffull;
    return (uint32_t)x;
}

// §1 grid transform
struct GridXf {
    float bmin[3];
    float E;
    float Nf;
    int N;
    int logN;
};

__device__ __forceinline__ float to_grid(const GridXf& g, int a, float p) {
    float t = p - g.bmin[a];
    t = t / g.E;
    return t * g.Nf;
}
__device__ __forceinline__ float to_grid_len(const GridXf& g, float r) {
    float t = r / g.E;
    return t * g.Nf;
}

// Shard filter: keys whose top cell (key >> shift) lies in [lo, hi) are emitted.
struct Shard {
    int shift;          // 3 * (logN - T)
    uint64_t cell_lo, cell_hi;
};

// Does the voxel box [e0, e1] (clamped to the grid) touch a top cell of the shard? Lets the
// emit kernels skip primitives that have no key in this rank's Morton range (their keys would
// all be filtered anyway), so per-rank emit work shrinks with the shard.
__device__ __forceinline__ bool box_in_shard(const int64_t* e0, const int64_t* e1, const Shard& sh) {
    const int s = sh.shift / 3;
    const int64_t c0x = e0[0] >> s, c1x = e1[0] >> s, c0y = e0[1] >> s, c1y = e1[1] >> s;
    const int64_t c0z = e0[2] >> s, c1z = e1[2] >> s;
    for (int64_t cz = c0z; cz <= c1z; cz++)
        for (int64_t cy = c0y; cy <= c1y; cy++)
            for (int64_t cx = c0x; cx <= c1x; cx++) {
                const uint64_t m = morton3((uint32_t)cx, (uint32_t)cy, (uint32_t)cz);
                if (m >= sh.cell_lo && m < sh.cell_hi) return true;
            }
    return false;
}

// Pair bins: Morton cells of 2^Lb voxels per edge (bin id = key >> shift, shift = 3 Lb).
// Each bin owns the pair slots [off[b], off[b+1]) -- its exact candidate count, an upper
// bound on its keys -- and cnt[b] pairs are appended there by the emit kernels.
struct Bins {
    int shift;
    const unsigned long long* off;   // [nb + 1]
    unsigned* cnt;                   // [nb]
};

// Appends the emitting lanes' pairs to their bins: lanes with the same bin share one atomic
// (warp match), and get consecutive slots. Must be called by the whole warp.
__device__ __forceinline__ void append_binned(bool emit, uint64_t mkey, uint64_t val, int lane, const Bins& bins,
                                              uint64_t* __restrict__ keys, uint64_t* __restrict__ vals,
                                              unsigned* __restrict__ flags) {
    const unsigned long long bk = emit ? (mkey >> bins.shift) : ~0ull;
    const unsigned m = __match_any_sync(0xffffffffu, bk);
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (emit && lane == leader) base = bins.off[bk] + atomicAdd(&bins.cnt[bk], (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (emit) {
        const uint64_t pos = base + __popc(m & ((1u << lane) - 1u));
        if (pos < bins.off[bk + 1]) {
            keys[pos] = mkey;
            vals[pos] = val;
        } else {
            atomicOr(flags, VOX_EFLAG_OVERFLOW);
        }
    }
}

// §13 sub-voxel density: index of `key` in a sorted key array (-1 if absent)
__device__ __forceinline__ long long find_key(const uint64_t* __restrict__ keys, uint64_t n, uint64_t key) {
    long long lo = 0, hi = (long long)n - 1;
    while (lo <= hi) {
        const long long mid = (lo + hi) >> 1;
        const uint64_t k = keys[mid];
        if (k == key) return mid;
        if (k < key) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

// ---------------------------------------------------------------- host-side state

// A level as the build leaves it: keys, exact accumulators and (levels >= 1) lobes. The fp32
// views (mass, m6, cl) are not written by the build; they are produced from the accumulators
// on demand (ensure_f32 / launch_finalize) when a caller reads the level.
struct Level {
    uint64_t n = 0;
    uint64_t* key = nullptr;
    long long* acc = nullptr;   // [n][7]
    uint8_t* ncl = nullptr;     // [n]       (levels >= 1)
    long long* clacc = nullptr; // [n][K][7] (levels >= 1); slots q >= ncl are undefined (never read)
    float* mass = nullptr;      // [n]        fp32 view, valid iff f32
    float* m6 = nullptr;        // [n][6]     fp32 view, valid iff f32
    float* cl = nullptr;        // [n][K][7]  fp32 view (levels >= 1), valid iff f32
    bool f32 = false;
};

enum CtxState { ST_CREATED = 0, ST_VOXELIZED = 1, ST_LOD = 2 };

// Per-stage CUDA-event timing without host syncs: begin/end events are recorded on the ctx
// stream and resolved in vox_stats_get.
struct StageTimer {
    cudaEvent_t open = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> done;
    double ms = 0.0;
};

}  // namespace vox

struct vox_ctx {
    vox::GridXf g;
    cudaStream_t stream = nullptr;
    int rank = 0, world = 1, T = 0;
    uint32_t K = 3;
    uint64_t max_bytes = 0;
    uint64_t part_cand = 3ull << 30;   // candidates per Morton part of one voxelize call
    int profile = 0;
    int state = vox::ST_CREATED;
    int built = 0;
    int imported_level = -1;
    bool plan_fixed = false;
    uint64_t cell_lo = 0, cell_hi = 0;
    vox::Level lv[VOX_MAX_LEVELS];
    unsigned int* d_flags = nullptr;        // device error flags
    unsigned long long* d_lodwork = nullptr; // [3]: SGGX-H sigma evals, distance evals, hard parents (profile)
    std::vector<cudaEvent_t> ev_pool;       // recycled timing events (profile)
    unsigned long long* d_counter = nullptr; // pair cursor
    vox_stats st{};
    std::string err;
    unsigned long long* dmask[VOX_MAX_LEVELS] = {};   // §13 sub-voxel masks per level ([n][8]), lazily
    int dmask_levels = -1;                  // levels with valid masks (0 after vox_density_*)
    cudaEvent_t ev_level[VOX_MAX_LEVELS] = {};   // recorded when a level's key/mass/m6 are final
    bool ev_level_ok[VOX_MAX_LEVELS] = {};
    // recorded on the caller's stream after a vox_copy_level_async of the level: freeing or
    // replacing the level's arrays first makes the ctx stream wait on it (the arrays go back to
    // the stream-keyed block cache and would otherwise be reused under the pending copy)
    cudaEvent_t ev_read[VOX_MAX_LEVELS] = {};
    bool ev_read_pending[VOX_MAX_LEVELS] = {};
    int dev = 0;                            // device of the ctx (event pool key)
    void* h_map = nullptr;                  // host-mapped pinned block for small readbacks
    void* d_map = nullptr;                  // its device alias
    int samp_n = 0;                         // samples per piece / triangle budget of the call (§12)
    const unsigned* samp_amax = nullptr;    // device max triangle area bits of the call (§12)
    int dmode = 0;                          // 0 sigma distance, 1 histogram distance (§10)
    int hist_n = 5000;                      // samples per histogram (§10)
    float* d_hist_u = nullptr;              // [3][N] sample table (SoA); process-wide, not owned
    uint32_t* d_hist_pg = nullptr;          // [124][32] (gap << 8) | cell of each slice step (transposed)
    // stage timers (profile = 1)
    vox::StageTimer t_bound, t_emit, t_sort, t_reduce, t_merge, t_lodscan, t_lod, t_vox, t_lodall, t_prep, t_quad, t_half, t_warp, t_encode, t_density;
};

namespace vox {

// allocation helpers (stream-ordered)
cudaError_t dalloc(vox_ctx* c, void** p, size_t bytes);
cudaError_t ssync(vox_ctx* c);   // cudaStreamSynchronize with host-time accounting
struct ReadItem {
    void* dst;
    const void* src;
    size_t bytes;
};
// small device->host reads through host-mapped memory (no copy engine), then a stream sync
cudaError_t readback(vox_ctx* c, std::initializer_list<ReadItem> items);
void dfree(vox_ctx* c, void* p);
void vox_trim_stream(cudaStream_t s);   // release the allocation cache of a stream
void free_level(vox_ctx* c, Level& L);
void timer_begin(vox_ctx* c, StageTimer& t);
void timer_end(vox_ctx* c, StageTimer& t);

// ---------------------------------------------------------------- kernel launchers

// fibers (k_fiber.cu)
cudaError_t launch_fiber_bound(vox_ctx* c, const float* seg, const float* rad, uint64_t S,
                               unsigned long long* cellW, int cell_log2);
cudaError_t launch_fiber_emit(vox_ctx* c, const float* seg, const float* rad, uint64_t S, Shard sh, Bins bins,
                              uint64_t* keys, uint64_t* vals, float4* ptab);
// triangles (k_tri.cu)
cudaError_t launch_tri_bound(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, unsigned long long* cellW,
                             int cell_log2);
cudaError_t launch_tri_emit(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, Shard sh, Bins bins,
                            uint64_t* keys, uint64_t* vals, float4* ptab);
// binned reduce (k_reduce.cu): per-bin pair lists -> new leaf set merged into lv[0]
struct LeafSet {
    uint64_t* key = nullptr;
    long long* acc = nullptr;
    uint64_t n = 0;
};
vox_status reduce_bins(vox_ctx* c, const uint64_t* keys, const uint64_t* vals, Bins bins, uint64_t nb,
                       const float4* ptab, LeafSet& out);
// merges a new leaf set into lv[0] (concatenation when its keys follow, exact sums otherwise)
vox_status merge_into_leaf(vox_ctx* c, uint64_t* nkey, long long* nacc, uint64_t V);
// per-call helpers (k_reduce.cu)
vox_status bin_topcells(vox_ctx* c, const unsigned long long* Wb, int Lb, std::vector<uint64_t>& WT);
vox_status bin_offsets(vox_ctx* c, const unsigned long long* Wb, int Lb, unsigned long long** off_out,
                       uint64_t* cap_out);
// single-pass exclusive scans, decoupled look-back (k_scan.cu)
cudaError_t scan_excl_u64(vox_ctx* c, const unsigned long long* in, unsigned long long* out, uint64_t n);
cudaError_t scan_excl_u32(vox_ctx* c, const unsigned* in, unsigned* out, uint64_t n);
cudaError_t scan_bin_caps(vox_ctx* c, const unsigned long long* Wb, uint64_t nb, int gshift, uint64_t lo, uint64_t hi,
                          unsigned long long* off);
cudaError_t scan_run_heads(vox_ctx* c, const uint64_t* key, uint64_t n, uint32_t* start, uint64_t* pkey,
                           uint32_t* total);
// LoD (k_lod.cu)
vox_status build_level(vox_ctx* c, int l);
void upload_theta(vox_ctx* c);
// histogram distance (k_hist.cu)
void host_hist_tables(int N, std::vector<float>& u, std::vector<uint8_t>& permT, std::vector<uint32_t>& gapT);
cudaError_t upload_hist_tables(vox_ctx* c);
// sampling front end (k_sample.cu)
cudaError_t launch_spline_bound(vox_ctx* c, const float* ctrl, const float* rad, uint64_t S, int n,
                                unsigned long long* cellW, int bin_log2);
cudaError_t launch_spline_emit(vox_ctx* c, const float* ctrl, const float* rad, uint64_t S, int n, Shard sh,
                               Bins bins, uint64_t* keys, uint64_t* vals, float4* ptab);
cudaError_t launch_tris_bound(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, int budget,
                              unsigned* amax_bits, unsigned long long* cellW, int bin_log2);
cudaError_t launch_tris_emit(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, int budget,
                             const unsigned* amax_bits, Shard sh, Bins bins, uint64_t* keys, uint64_t* vals,
                             float4* ptab);
// sub-voxel density (k_fiber.cu, k_tri.cu, k_density.cu)
cudaError_t launch_fiber_density(vox_ctx* c, const float* seg, const float* rad, uint64_t S);
cudaError_t launch_tri_density(vox_ctx* c, const float* tri, uint64_t T);
cudaError_t launch_density_down(vox_ctx* c, int level);   // masks of `level` from level - 1
cudaError_t launch_density_stats(vox_ctx* c, int level, float* occ, float* axis);
// compact form (k_encode.cu)
cudaError_t launch_encode(vox_ctx* c, const Level& L, int leaf, uint8_t* out6, uint8_t* cl6, uint8_t* flags);
cudaError_t launch_sggxh_hist(vox_ctx* c, int K, const uint32_t* list, const unsigned* counts, const Level& C,
                              int leaf, const uint32_t* start, Level& P);
void host_theta(float theta[32][3], float coef[32][6]);
// fp32 views of a level from its accumulators (k_lod.cu): writes whichever of mass / m6 / cl
// is non-null, for n records, on stream s
cudaError_t launch_finalize(vox_ctx* c, cudaStream_t s, uint64_t n, const long long* acc, const uint8_t* ncl,
                            const long long* clacc, float* mass, float* m6, float* cl);
// allocates and fills the level's fp32 views once (ctx stream); no-op when already valid
vox_status ensure_f32(vox_ctx* c, int level);
// multi-GPU records (k_lod.cu)
uint64_t record_bytes(uint32_t K);
cudaError_t launch_pack(vox_ctx* c, int level, void* buf);
vox_status unpack_level(vox_ctx* c, int level, const void* buf, uint64_t n);

}  // namespace vox
