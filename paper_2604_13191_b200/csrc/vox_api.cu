// vox_api.cu -- the C ABI (include/vox.h): validation, the ctx state machine, stream-ordered
// allocation, the per-call pipeline (bound -> plan/capacity -> emit -> sort/reduce -> merge)
// and the multi-GPU level export/import.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <chrono>
#include <map>
#include <set>
#include <unordered_map>
#include <mutex>
#include <new>

#include "vox_internal.cuh"

namespace vox {

double host_ms_since(const std::chrono::steady_clock::time_point& t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Device memory: a process-wide caching allocator (best fit within 2x, per stream). Blocks
// freed by a call go back to the cache and are reused by later calls on the same stream, so
// stream order makes reuse safe; cudaMallocAsync is only hit on a cache miss (its pool showed
// multi-10-ms stalls when the same sizes were requested step after step). vox_trim releases.
struct CachedBlock {
    cudaStream_t stream;
    size_t bytes;
};
static std::mutex g_mem_mu;
static std::multimap<std::pair<cudaStream_t, size_t>, void*> g_free;   // (stream, bytes) -> ptr
static std::unordered_map<void*, CachedBlock> g_live;

static size_t round_bytes(size_t b) {
    if (b <= 4096) return 4096;
    if (b <= (1u << 20)) {   // powers of two up to 1 MiB
        size_t r = 4096;
        while (r < b) r <<= 1;
        return r;
    }
    return (b + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);   // 2 MiB granularity
}

// stream-ordered allocation on the ctx stream; freed blocks are cached per stream (a block is
// only handed out again on the stream that used it)
cudaError_t dalloc(vox_ctx* c, void** p, size_t bytes) {
    cudaStream_t s = c->stream;
    *p = nullptr;
    const size_t want = round_bytes((bytes ? bytes : 16) + 64);   // >= 64 B slack (bulk-copy tails)
    const auto t0 = std::chrono::steady_clock::now();
    {
        std::lock_guard<std::mutex> lk(g_mem_mu);
        auto it = g_free.lower_bound({s, want});
        if (it != g_free.end() && it->first.first == s && it->first.second <= 2 * want) {
            *p = it->second;
            g_live[*p] = CachedBlock{s, it->first.second};
            g_free.erase(it);
        }
    }
    cudaError_t e = cudaSuccess;
    if (!*p) {
        e = cudaMallocAsync(p, want, s);
        if (e == cudaErrorMemoryAllocation) {
            // release the cached blocks of this stream, return the pool's unused memory, retry
            cudaGetLastError();
            vox_trim_stream(s);
            cudaStreamSynchronize(s);
            int dev = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
                cudaMemPoolTrimTo(pool, 0);
            e = cudaMallocAsync(p, want, s);
        }
        if (e == cudaSuccess) {
            std::lock_guard<std::mutex> lk(g_mem_mu);
            g_live[*p] = CachedBlock{s, want};
        }
    }
    c->st.host_ms_alloc += host_ms_since(t0);
    return e;
}

void dfree(vox_ctx* c, void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_mem_mu);
    auto it = g_live.find(p);
    if (it == g_live.end()) {   // not ours (should not happen)
        cudaFreeAsync(p, c->stream);
        return;
    }
    g_free.insert({{it->second.stream, it->second.bytes}, p});
    g_live.erase(it);
}

void vox_trim_stream(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_mem_mu);
    for (auto it = g_free.begin(); it != g_free.end();) {
        if (it->first.first == s) {
            cudaFreeAsync(it->second, s);
            it = g_free.erase(it);
        } else {
            ++it;
        }
    }
}

cudaError_t ssync(vox_ctx* c) {
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaStreamSynchronize(c->stream);
    c->st.host_ms_sync += host_ms_since(t0);
    return e;
}

// Small device->host reads (counts, flags) without the copy engines: a one-block kernel
// copies the words into host-mapped pinned memory, then the ctx stream is synchronised. A
// cudaMemcpyAsync would queue behind large D2H transfers the caller may have in flight on
// another stream (vox_copy_level_async) and serialise the build with them.
__global__ void k_peek(const unsigned* __restrict__ src, unsigned* __restrict__ dst, int nwords) {
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = src[i];
}

static std::mutex g_map_mu;
static std::map<int, std::vector<std::pair<void*, void*>>> g_map_pool;   // per device: (host, device alias)
constexpr size_t MAP_BYTES = 64 * 1024;

static cudaError_t acquire_mapped(vox_ctx* c) {
    if (c->h_map) return cudaSuccess;
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        std::vector<std::pair<void*, void*>>& pool = g_map_pool[c->dev];
        if (!pool.empty()) {
            c->h_map = pool.back().first;
            c->d_map = pool.back().second;
            pool.pop_back();
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaHostAlloc(&c->h_map, MAP_BYTES, cudaHostAllocMapped);
    if (e != cudaSuccess) return e;
    return cudaHostGetDevicePointer(&c->d_map, c->h_map, 0);
}

static void release_mapped(vox_ctx* c) {
    if (!c->h_map) return;
    std::lock_guard<std::mutex> lk(g_map_mu);
    g_map_pool[c->dev].push_back({c->h_map, c->d_map});
    c->h_map = c->d_map = nullptr;
}

cudaError_t readback(vox_ctx* c, std::initializer_list<ReadItem> items) {
    cudaError_t e = acquire_mapped(c);
    if (e != cudaSuccess) return e;
    size_t off = 0;
    for (const ReadItem& it : items) {
        const size_t words = (it.bytes + 3) / 4;
        if ((off + words) * 4 > MAP_BYTES) return cudaErrorInvalidValue;
        k_peek<<<1, 256, 0, c->stream>>>(reinterpret_cast<const unsigned*>(it.src),
                                         reinterpret_cast<unsigned*>(c->d_map) + off, (int)words);
        off += words;
    }
    c->st.launches += items.size();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = ssync(c);
    if (e != cudaSuccess) return e;
    off = 0;
    for (const ReadItem& it : items) {
        std::memcpy(it.dst, reinterpret_cast<const unsigned*>(c->h_map) + off, it.bytes);
        off += (it.bytes + 3) / 4;
    }
    return cudaSuccess;
}

void free_level(vox_ctx* c, Level& L) {
    if (&L >= c->lv && &L < c->lv + VOX_MAX_LEVELS) {
        const int l = (int)(&L - c->lv);
        if (c->ev_read_pending[l]) {   // an async copy of this level may still be reading it
            cudaStreamWaitEvent(c->stream, c->ev_read[l], 0);
            c->ev_read_pending[l] = false;
        }
    }
    dfree(c, L.key); dfree(c, L.acc); dfree(c, L.ncl); dfree(c, L.clacc);
    dfree(c, L.mass); dfree(c, L.m6); dfree(c, L.cl);
    L = Level();
}

// Timing events are recycled process-wide: creating events costs tens of microseconds,
// which would add up over the ~200 stage events of one voxelize + LoD build.
static std::mutex g_ev_mu;
static std::map<int, std::vector<cudaEvent_t>> g_ev_pool;   // per device: events are device-bound

static cudaEvent_t event_get(vox_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    {
        std::lock_guard<std::mutex> lk(g_ev_mu);
        std::vector<cudaEvent_t>& pool = g_ev_pool[c->dev];
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return e;
}

// Timing is best effort: a failed event creation or record drops the sample and clears the
// error, so it can never surface later as a launcher's VOX_ERR_CUDA.
void timer_begin(vox_ctx* c, StageTimer& t) {
    if (!c->profile) return;
    t.open = event_get(c);
    if (t.open && cudaEventRecord(t.open, c->stream) != cudaSuccess) {
        cudaGetLastError();
        c->ev_pool.push_back(t.open);
        t.open = nullptr;
    }
}

void timer_end(vox_ctx* c, StageTimer& t) {
    if (!c->profile || !t.open) return;
    cudaEvent_t b = event_get(c);
    if (!b || cudaEventRecord(b, c->stream) != cudaSuccess) {
        cudaGetLastError();
        c->ev_pool.push_back(t.open);
        if (b) c->ev_pool.push_back(b);
        t.open = nullptr;
        return;
    }
    t.done.emplace_back(t.open, b);
    t.open = nullptr;
}

static double timer_flush(vox_ctx* c, StageTimer& t) {
    for (auto& pr : t.done) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) t.ms += ms;
        c->ev_pool.push_back(pr.first);
        c->ev_pool.push_back(pr.second);
    }
    t.done.clear();
    return t.ms;
}

}  // namespace vox

using namespace vox;

#define CKS(x)                                                         \
    do {                                                               \
        cudaError_t e_ = (x);                                          \
        if (e_ != cudaSuccess) {                                       \
            c->err = std::string(#x) + ": " + cudaGetErrorString(e_);  \
            return e_ == cudaErrorMemoryAllocation ? VOX_ERR_OOM : VOX_ERR_CUDA; \
        }                                                              \
    } while (0)

static vox_status ensure_dev(vox_ctx* c) {
    if (c->d_flags) return VOX_OK;
    // keep freed stream-ordered allocations in the pool across calls (no re-mapping per step)
    int dev = 0;
    cudaMemPool_t pool;
    CKS(cudaGetDevice(&dev));
    CKS(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    CKS(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // no hidden cross-stream waits: memory freed on an async-copy stream (the fp32-view
    // scratch of vox_copy_level_async) must not be handed to the ctx stream by making it wait
    // for that stream -- the build would stall behind the D2H. Completed frees are still reused.
    int no_dep = 0;
    CKS(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no_dep));
    CKS(cudaMallocAsync((void**)&c->d_flags, 16, c->stream));
    CKS(cudaMallocAsync((void**)&c->d_counter, 16, c->stream));
    CKS(cudaMallocAsync((void**)&c->d_lodwork, 32, c->stream));
    CKS(cudaMemsetAsync(c->d_lodwork, 0, 32, c->stream));
    upload_theta(c);
    if (c->dmode == 1) CKS(upload_hist_tables(c));
    CKS(cudaGetLastError());
    return VOX_OK;
}

extern "C" {

const char* vox_status_str(vox_status s) {
    switch (s) {
        case VOX_OK: return "VOX_OK";
        case VOX_ERR_INVALID_ARG: return "VOX_ERR_INVALID_ARG";
        case VOX_ERR_DEGENERATE_BBOX: return "VOX_ERR_DEGENERATE_BBOX";
        case VOX_ERR_STATE: return "VOX_ERR_STATE";
        case VOX_ERR_OOM: return "VOX_ERR_OOM";
        case VOX_ERR_CAPACITY: return "VOX_ERR_CAPACITY";
        case VOX_ERR_CUDA: return "VOX_ERR_CUDA";
        case VOX_ERR_LEVEL: return "VOX_ERR_LEVEL";
        case VOX_ERR_COMM: return "VOX_ERR_COMM";
    }
    return "VOX_ERR_UNKNOWN";
}

const char* vox_last_error(vox_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

vox_status vox_create(vox_ctx** out, uint32_t grid_res, const float bbox[6], const vox_options* opt) {
    VOX_RANGE("vox_create");
    if (!out || !bbox) return VOX_ERR_INVALID_ARG;
    *out = nullptr;
    if (grid_res < 2 || grid_res > 8192 || (grid_res & (grid_res - 1))) return VOX_ERR_INVALID_ARG;
    float e[3];
    for (int a = 0; a < 3; a++) {
        if (!std::isfinite(bbox[a]) || !std::isfinite(bbox[3 + a])) return VOX_ERR_DEGENERATE_BBOX;
        e[a] = bbox[3 + a] - bbox[a];
        if (!(e[a] > 0.0f)) return VOX_ERR_DEGENERATE_BBOX;
    }
    vox_options o{};
    if (opt) o = *opt;
    int logN = 0;
    while ((1u << logN) < grid_res) logN++;
    if (o.world == 0) o.world = 1;
    if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return VOX_ERR_INVALID_ARG;
    if (o.top_depth == 0) o.top_depth = std::min(4, logN);
    if (o.top_depth < 1 || o.top_depth > std::min(5, logN)) return VOX_ERR_INVALID_ARG;
    if (o.k == 0) o.k = 3;
    if (o.k > VOX_MAX_K) return VOX_ERR_INVALID_ARG;
    if (o.n_slices != 0 && o.n_slices != VOX_SLICES) return VOX_ERR_INVALID_ARG;
    if (o.distance_mode < 0 || o.distance_mode > 1) return VOX_ERR_INVALID_ARG;
    if (o.hist_samples == 0) o.hist_samples = 5000;
    if (o.hist_samples < 32 || o.hist_samples > 8160) return VOX_ERR_INVALID_ARG;
    if (o.part_candidates == 0) o.part_candidates = 3ull << 30;
    if (o.part_candidates > (3ull << 30)) return VOX_ERR_INVALID_ARG;
    vox_ctx* c = new (std::nothrow) vox_ctx();
    if (!c) return VOX_ERR_OOM;
    for (int a = 0; a < 3; a++) c->g.bmin[a] = bbox[a];
    c->g.E = pmax(pmax(e[0], e[1]), e[2]);
    c->g.N = (int)grid_res;
    c->g.Nf = (float)grid_res;
    c->g.logN = logN;
    c->stream = (cudaStream_t)o.stream;
    c->rank = o.rank;
    c->world = o.world;
    c->T = o.top_depth;
    c->K = o.k;
    c->max_bytes = o.max_bytes;
    c->profile = o.profile;
    c->dmode = o.distance_mode;
    c->hist_n = (int)o.hist_samples;
    c->part_cand = o.part_candidates;
    c->built = 0;
    c->st.top_depth = (uint32_t)c->T;
    if (cudaGetDevice(&c->dev) != cudaSuccess) {
        cudaGetLastError();
        c->dev = 0;
    }
    *out = c;
    return VOX_OK;
}

static uint64_t ncells_of(const vox_ctx* c) { return 1ull << (3 * c->T); }

vox_status vox_plan_shards(const uint64_t* w, uint64_t ncells, int world, uint64_t* bounds) {
    if (!w || !bounds || world < 1 || ncells == 0) return VOX_ERR_INVALID_ARG;
    unsigned __int128 total = 0;
    for (uint64_t x = 0; x < ncells; x++) total += w[x];
    bounds[0] = 0;
    bounds[world] = ncells;
    if (total == 0) {
        for (int r = 1; r < world; r++) bounds[r] = (uint64_t)((unsigned __int128)ncells * r / world);
        return VOX_OK;
    }
    // rank r starts at the first cell whose exclusive prefix weight reaches r/world of the total
    unsigned __int128 pre = 0;
    uint64_t x = 0;
    for (int r = 1; r < world; r++) {
        const unsigned __int128 target = total * (unsigned __int128)r;
        while (x < ncells && pre * (unsigned __int128)world < target) pre += w[x++];
        bounds[r] = x;
    }
    return VOX_OK;
}

// Common tail of the two voxelize entry points: bound (done), plan, capacity, emit, reduce.
typedef cudaError_t (*emit_fn)(vox_ctx*, const float*, const float*, uint64_t, Shard, Bins, uint64_t*, uint64_t*,
                               float4*);

// bins of 16^3 voxels (32^3 at 8192^3 to bound the bin arrays), never coarser than a top cell
static int bin_log2(const vox_ctx* c) { return std::min(c->g.logN >= 13 ? 5 : 4, c->g.logN - c->T); }
static uint64_t nbins_of(const vox_ctx* c) { return 1ull << (3 * (c->g.logN - bin_log2(c))); }

static void density_reset(vox_ctx* c);

static vox_status voxelize_common(vox_ctx* c, const float* a, const float* b, uint64_t n, unsigned long long* Wb,
                                  emit_fn emit, uint64_t nptab = 0) {
    density_reset(c);   // level 0 changes: sub-voxel masks must be recomputed (vox_density_*)
    if (nptab == 0) nptab = n;   // prim-table entries (one per sample for the spline front end)
    const uint64_t ncells = ncells_of(c), nb = nbins_of(c);
    const int Lb = bin_log2(c);
    unsigned fl = 0;
    CKS(readback(c, {{&fl, c->d_flags, 4}}));
    timer_end(c, c->t_bound);
    if (fl) {
        dfree(c, Wb);
        c->err = std::string("invalid input:") + ((fl & VOX_EFLAG_NONFINITE) ? " non-finite value" : "") +
                 ((fl & VOX_EFLAG_NEG_RADIUS) ? " negative radius" : "") +
                 ((fl & VOX_EFLAG_TOO_MANY_CAND) ? " segment with more than 2^24 candidate voxels" : "") +
                 ((fl & VOX_EFLAG_ZERO_DIR) ? " zero-norm dir" : "");
        return VOX_ERR_INVALID_ARG;
    }
    vox_status s;
    if (!c->plan_fixed) {
        if (c->world == 1) {
            c->cell_lo = 0;
            c->cell_hi = ncells;
        } else {
            std::vector<uint64_t> W;
            s = bin_topcells(c, Wb, Lb, W);
            if (s != VOX_OK) return s;
            std::vector<uint64_t> bounds(c->world + 1);
            vox_plan_shards(W.data(), ncells, c->world, bounds.data());
            c->cell_lo = bounds[c->rank];
            c->cell_hi = bounds[c->rank + 1];
        }
        c->plan_fixed = true;
        c->st.cell_lo = c->cell_lo;
        c->st.cell_hi = c->cell_hi;
    }
    // Parts: this rank's top-cell range, split (in Morton order) so that every part's candidate
    // count fits the 32-bit pair slots (and the part_candidates bound). Each part emits only its
    // keys (the shard filter; a primitive's S_p still sums all its keys) and its leaves follow
    // the previous part's in key order, so the parts' leaf sets are concatenated.
    const uint64_t lo0 = c->cell_lo, hi0 = c->cell_hi;
    std::vector<uint64_t> cuts = {lo0, hi0};
    unsigned long long* off1 = nullptr;   // offsets of the whole range, re-used by a single part
    uint64_t cap1 = 0;
    {
        s = bin_offsets(c, Wb, Lb, &off1, &cap1);
        if (s != VOX_OK) { dfree(c, Wb); return s; }
        c->st.candidates = cap1;
        if (cap1 > c->part_cand) {
            dfree(c, off1);
            off1 = nullptr;
            std::vector<uint64_t> W;
            s = bin_topcells(c, Wb, Lb, W);
            if (s != VOX_OK) { dfree(c, Wb); return s; }
            cuts = {lo0};
            uint64_t acc = 0;
            for (uint64_t x = lo0; x < hi0; x++) {
                if (W[x] >= (3ull << 30)) {   // one top cell must fit the 32-bit pair slots
                    dfree(c, Wb);
                    c->err = "a top cell with more than 3*2^30 candidate voxels: use a larger top_depth";
                    return VOX_ERR_CAPACITY;
                }
                if (acc > 0 && acc + W[x] > c->part_cand) {
                    cuts.push_back(x);
                    acc = 0;
                }
                acc += W[x];
            }
            cuts.push_back(hi0);
        }
    }
    c->st.pairs = 0;
    auto run_part = [&]() -> vox_status {
        unsigned long long* off = off1;
        uint64_t cap = cap1;
        vox_status r = VOX_OK;
        if (!off) {
            r = bin_offsets(c, Wb, Lb, &off, &cap);
            if (r != VOX_OK) return r;
        }
        off1 = nullptr;   // owned (and freed) by this part from here
        if (cap == 0) {
            dfree(c, off);
            return VOX_OK;
        }
        // estimate: pairs + per-bin scans + new leaf (<= cap voxels) + prim table + merge
        const uint64_t est = cap * 16 + nb * 24 + cap * 92 + nptab * 16 + c->lv[0].n * 92;
        if (c->max_bytes && est > c->max_bytes) {
            dfree(c, off);
            c->err = "estimated " + std::to_string(est) + " bytes exceed max_bytes";
            return VOX_ERR_CAPACITY;
        }
        uint64_t *keys = nullptr, *vals = nullptr;
        float4* ptab = nullptr;
        unsigned* bcnt = nullptr;
        auto release = [&]() {   // pair scratch, released before the leaf merge
            dfree(c, keys);
            dfree(c, vals);
            dfree(c, ptab);
            dfree(c, bcnt);
            dfree(c, off);
        };
        cudaError_t e = dalloc(c, (void**)&keys, cap * 8);
        if (e == cudaSuccess) e = dalloc(c, (void**)&vals, cap * 8);
        if (e == cudaSuccess) e = dalloc(c, (void**)&ptab, nptab * sizeof(float4));
        if (e == cudaSuccess) e = dalloc(c, (void**)&bcnt, nb * 4);
        if (e == cudaSuccess) e = cudaMemsetAsync(bcnt, 0, nb * 4, c->stream);
        if (e != cudaSuccess) {
            release();
            c->err = std::string("voxelize scratch: ") + cudaGetErrorString(e);
            return e == cudaErrorMemoryAllocation ? VOX_ERR_OOM : VOX_ERR_CUDA;
        }
        Shard sh;
        sh.shift = 3 * (c->g.logN - c->T);
        sh.cell_lo = c->cell_lo;
        sh.cell_hi = c->cell_hi;
        Bins bins;
        bins.shift = 3 * Lb;
        bins.off = off;
        bins.cnt = bcnt;
        timer_begin(c, c->t_emit);
        e = emit(c, a, b, n, sh, bins, keys, vals, ptab);
        timer_end(c, c->t_emit);
        if (e != cudaSuccess) {
            release();
            c->err = std::string("emit: ") + cudaGetErrorString(e);
            return VOX_ERR_CUDA;
        }
        LeafSet leaf;
        r = reduce_bins(c, keys, vals, bins, nb, ptab, leaf);
        unsigned fl2 = 0;
        e = r == VOX_OK ? readback(c, {{&fl2, c->d_flags, 4}}) : cudaSuccess;
        release();
        if (r != VOX_OK) return r;
        if (e != cudaSuccess) {
            c->err = std::string("readback: ") + cudaGetErrorString(e);
            return e == cudaErrorMemoryAllocation ? VOX_ERR_OOM : VOX_ERR_CUDA;
        }
        if (fl2 & VOX_EFLAG_OVERFLOW) {
            c->err = "internal: pair capacity overflow";
            return VOX_ERR_CUDA;
        }
        return merge_into_leaf(c, leaf.key, leaf.acc, leaf.n);
    };
    vox_status res = VOX_OK;
    for (size_t part = 0; part + 1 < cuts.size() && res == VOX_OK; part++) {
        c->cell_lo = cuts[part];
        c->cell_hi = cuts[part + 1];
        res = run_part();
    }
    c->cell_lo = lo0;
    c->cell_hi = hi0;
    dfree(c, Wb);
    if (res != VOX_OK) return res;
    c->st.voxels = c->lv[0].n;
    c->state = ST_VOXELIZED;
    return VOX_OK;
}

static cudaError_t emit_fibers(vox_ctx* c, const float* seg, const float* rad, uint64_t S, Shard sh, Bins bins,
                               uint64_t* keys, uint64_t* vals, float4* ptab) {
    return launch_fiber_emit(c, seg, rad, S, sh, bins, keys, vals, ptab);
}

static cudaError_t emit_tris(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, Shard sh, Bins bins,
                             uint64_t* keys, uint64_t* vals, float4* ptab) {
    return launch_tri_emit(c, tri, dirs, T, sh, bins, keys, vals, ptab);
}

vox_status vox_voxelize_fibers(vox_ctx* c, const float* segments, const float* radii, uint64_t S) {
    VOX_RANGE("vox_voxelize_fibers");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (c->state == ST_LOD) return VOX_ERR_STATE;
    if (S == 0) return VOX_OK;
    if (!segments || !radii || S >= (1ull << 32)) return VOX_ERR_INVALID_ARG;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    c->st.segments = S;
    timer_begin(c, c->t_vox);
    timer_begin(c, c->t_bound);
    const uint64_t nb = nbins_of(c);
    unsigned long long* cellW = nullptr;
    CKS(dalloc(c, (void**)&cellW, nb * 8));
    CKS(cudaMemsetAsync(cellW, 0, nb * 8, c->stream));
    CKS(cudaMemsetAsync(c->d_flags, 0, 4, c->stream));
    CKS(launch_fiber_bound(c, segments, radii, S, cellW, bin_log2(c)));
    s = voxelize_common(c, segments, radii, S, cellW, emit_fibers);
    timer_end(c, c->t_vox);
    return s;
}

vox_status vox_voxelize_triangles(vox_ctx* c, const float* tris, const float* dirs, uint64_t T) {
    VOX_RANGE("vox_voxelize_triangles");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (c->state == ST_LOD) return VOX_ERR_STATE;
    if (T == 0) return VOX_OK;
    if (!tris || T >= (1ull << 32)) return VOX_ERR_INVALID_ARG;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    c->st.segments = T;
    timer_begin(c, c->t_vox);
    timer_begin(c, c->t_bound);
    const uint64_t nb = nbins_of(c);
    unsigned long long* cellW = nullptr;
    CKS(dalloc(c, (void**)&cellW, nb * 8));
    CKS(cudaMemsetAsync(cellW, 0, nb * 8, c->stream));
    CKS(cudaMemsetAsync(c->d_flags, 0, 4, c->stream));
    CKS(launch_tri_bound(c, tris, dirs, T, cellW, bin_log2(c)));
    s = voxelize_common(c, tris, dirs, T, cellW, emit_tris);
    timer_end(c, c->t_vox);
    return s;
}

// ---------------------------------------------------------------- the paper's sampling front end (§12)
static cudaError_t emit_splines(vox_ctx* c, const float* ctrl, const float* rad, uint64_t S, Shard sh, Bins bins,
                                uint64_t* keys, uint64_t* vals, float4* ptab) {
    return launch_spline_emit(c, ctrl, rad, S, c->samp_n, sh, bins, keys, vals, ptab);
}

static cudaError_t emit_sampled_tris(vox_ctx* c, const float* tri, const float* dirs, uint64_t T, Shard sh,
                                     Bins bins, uint64_t* keys, uint64_t* vals, float4* ptab) {
    return launch_tris_emit(c, tri, dirs, T, c->samp_n, c->samp_amax, sh, bins, keys, vals, ptab);
}

vox_status vox_sample_splines(vox_ctx* c, const float* ctrl, const float* radii, uint64_t S, uint32_t n) {
    VOX_RANGE("vox_sample_splines");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (c->state == ST_LOD) return VOX_ERR_STATE;
    if (S == 0) return VOX_OK;
    if (!ctrl || !radii || n < 1 || n > 65536 || S * (uint64_t)n >= (1ull << 32)) return VOX_ERR_INVALID_ARG;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    c->st.segments = S;
    timer_begin(c, c->t_vox);
    timer_begin(c, c->t_bound);
    const uint64_t nb = nbins_of(c);
    unsigned long long* cellW = nullptr;
    CKS(dalloc(c, (void**)&cellW, nb * 8));
    CKS(cudaMemsetAsync(cellW, 0, nb * 8, c->stream));
    CKS(cudaMemsetAsync(c->d_flags, 0, 4, c->stream));
    CKS(launch_spline_bound(c, ctrl, radii, S, (int)n, cellW, bin_log2(c)));
    c->samp_n = (int)n;
    s = voxelize_common(c, ctrl, radii, S, cellW, emit_splines, S * (uint64_t)n);
    timer_end(c, c->t_vox);
    return s;
}

vox_status vox_sample_triangles(vox_ctx* c, const float* tris, const float* dirs, uint64_t T, uint32_t budget) {
    VOX_RANGE("vox_sample_triangles");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (c->state == ST_LOD) return VOX_ERR_STATE;
    if (T == 0) return VOX_OK;
    if (!tris || budget < 1 || budget > 65536 || T >= (1ull << 32)) return VOX_ERR_INVALID_ARG;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    c->st.segments = T;
    timer_begin(c, c->t_vox);
    timer_begin(c, c->t_bound);
    const uint64_t nb = nbins_of(c);
    unsigned long long* cellW = nullptr;
    CKS(dalloc(c, (void**)&cellW, nb * 8));
    CKS(cudaMemsetAsync(cellW, 0, nb * 8, c->stream));
    CKS(cudaMemsetAsync(c->d_flags, 0, 4, c->stream));
    unsigned* amax = nullptr;
    CKS(dalloc(c, (void**)&amax, 16));
    CKS(launch_tris_bound(c, tris, dirs, T, (int)budget, amax, cellW, bin_log2(c)));
    c->samp_n = (int)budget;
    c->samp_amax = amax;
    s = voxelize_common(c, tris, dirs, T, cellW, emit_sampled_tris);
    c->samp_amax = nullptr;
    dfree(c, amax);
    timer_end(c, c->t_vox);
    return s;
}

vox_status vox_voxelize_fibers_host(vox_ctx* c, const float* segments, const float* radii, uint64_t S) {
    VOX_RANGE("vox_voxelize_fibers_host");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (c->state == ST_LOD) return VOX_ERR_STATE;
    if (S == 0) return VOX_OK;
    if (!segments || !radii) return VOX_ERR_INVALID_ARG;
    float *ds = nullptr, *dr = nullptr;
    CKS(dalloc(c, (void**)&ds, S * 24));
    CKS(dalloc(c, (void**)&dr, S * 4));
    CKS(cudaMemcpyAsync(ds, segments, S * 24, cudaMemcpyHostToDevice, c->stream));
    CKS(cudaMemcpyAsync(dr, radii, S * 4, cudaMemcpyHostToDevice, c->stream));
    vox_status s = vox_voxelize_fibers(c, ds, dr, S);
    dfree(c, ds);
    dfree(c, dr);
    return s;
}

vox_status vox_voxelize_triangles_host(vox_ctx* c, const float* tris, const float* dirs, uint64_t T) {
    VOX_RANGE("vox_voxelize_triangles_host");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (c->state == ST_LOD) return VOX_ERR_STATE;
    if (T == 0) return VOX_OK;
    if (!tris) return VOX_ERR_INVALID_ARG;
    float *dt = nullptr, *dd = nullptr;
    CKS(dalloc(c, (void**)&dt, T * 36));
    CKS(cudaMemcpyAsync(dt, tris, T * 36, cudaMemcpyHostToDevice, c->stream));
    if (dirs) {
        CKS(dalloc(c, (void**)&dd, T * 12));
        CKS(cudaMemcpyAsync(dd, dirs, T * 12, cudaMemcpyHostToDevice, c->stream));
    }
    vox_status s = vox_voxelize_triangles(c, dt, dd, T);
    dfree(c, dt);
    dfree(c, dd);
    return s;
}

vox_status vox_build_lod(vox_ctx* c, uint32_t levels) {
    VOX_RANGE("vox_build_lod");
    if (!c) return VOX_ERR_INVALID_ARG;
    if ((int)levels > c->g.logN) return VOX_ERR_LEVEL;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    int limit = (int)levels;
    const int Lt = c->g.logN - c->T;
    if (c->world > 1 && c->imported_level < 0 && limit > Lt) limit = Lt;
    timer_begin(c, c->t_lodall);
    for (int l = c->built + 1; l <= limit; l++) {
        s = build_level(c, l);
        if (s != VOX_OK) return s;
        c->built = l;
    }
    timer_end(c, c->t_lodall);
    c->state = ST_LOD;
    return VOX_OK;
}

vox_status vox_built_levels(vox_ctx* c, uint32_t* out) {
    if (!c || !out) return VOX_ERR_INVALID_ARG;
    *out = (uint32_t)c->built;
    return VOX_OK;
}

vox_status vox_level_size(vox_ctx* c, uint32_t level, uint64_t* out) {
    if (!c || !out) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    *out = c->lv[level].n;
    return VOX_OK;
}

vox_status vox_read_level(vox_ctx* c, uint32_t level, vox_level_view* out) {
    VOX_RANGE("vox_read_level");
    if (!c || !out) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    vox_status s = ensure_f32(c, (int)level);   // the build keeps only the exact accumulators
    if (s != VOX_OK) return s;
    const Level& L = c->lv[level];
    out->n = L.n;
    out->key = L.key;
    out->mass = L.mass;
    out->m6 = L.m6;
    out->acc = reinterpret_cast<const int64_t*>(L.acc);
    out->ncl = level == 0 ? nullptr : L.ncl;
    out->cl = level == 0 ? nullptr : L.cl;
    return VOX_OK;
}

// a leaf's single lobe is (mass, M) iff mass > 0 (D17)
__global__ void k_leaf_lobes(uint64_t n, const long long* __restrict__ acc, int K, uint8_t* __restrict__ ncl,
                             float* __restrict__ cl) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const bool has = acc[7 * v] > 0;
        if (ncl) ncl[v] = has ? 1 : 0;
        if (cl) {
            for (int q = 0; q < K; q++)
                for (int e = 0; e < 7; e++) cl[(v * K + q) * 7 + e] = (q == 0 && has) ? deq32(acc[7 * v + e]) : 0.0f;
        }
    }
}

// ---------------------------------------------------------------- §13 sub-voxel density
static void density_reset(vox_ctx* c) {
    for (int l = 0; l < VOX_MAX_LEVELS; l++)
        if (c->dmask[l]) {
            dfree(c, c->dmask[l]);
            c->dmask[l] = nullptr;
        }
    c->dmask_levels = -1;
}

static vox_status density_prepare(vox_ctx* c) {
    if (c->state == ST_CREATED || c->built < 0) return VOX_ERR_STATE;
    for (int l = 1; l < VOX_MAX_LEVELS; l++)   // lower-level masks change: rebuild upper ones lazily
        if (c->dmask[l]) {
            dfree(c, c->dmask[l]);
            c->dmask[l] = nullptr;
        }
    if (!c->dmask[0]) {
        const uint64_t n0 = c->lv[0].n;
        CKS(dalloc(c, (void**)&c->dmask[0], (n0 ? n0 : 1) * 64));
        CKS(cudaMemsetAsync(c->dmask[0], 0, (n0 ? n0 : 1) * 64, c->stream));
    }
    c->dmask_levels = 0;
    return VOX_OK;
}

vox_status vox_density_fibers(vox_ctx* c, const float* segments, const float* radii, uint64_t S) {
    VOX_RANGE("vox_density_fibers");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (S && (!segments || !radii)) return VOX_ERR_INVALID_ARG;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    s = density_prepare(c);
    if (s != VOX_OK) return s;
    if (S == 0 || c->lv[0].n == 0) return VOX_OK;
    timer_begin(c, c->t_density);
    CKS(launch_fiber_density(c, segments, radii, S));
    timer_end(c, c->t_density);
    return VOX_OK;
}

vox_status vox_density_triangles(vox_ctx* c, const float* tris, uint64_t T) {
    VOX_RANGE("vox_density_triangles");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (T && !tris) return VOX_ERR_INVALID_ARG;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    s = density_prepare(c);
    if (s != VOX_OK) return s;
    if (T == 0 || c->lv[0].n == 0) return VOX_OK;
    timer_begin(c, c->t_density);
    CKS(launch_tri_density(c, tris, T));
    timer_end(c, c->t_density);
    return VOX_OK;
}

vox_status vox_density_level(vox_ctx* c, uint32_t level, float* occ, float* axis, uint64_t* masks) {
    VOX_RANGE("vox_density_level");
    if (!c) return VOX_ERR_INVALID_ARG;
    if (c->dmask_levels < 0) return VOX_ERR_STATE;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    if (c->world > 1 && (int)level > c->g.logN - c->T) return VOX_ERR_STATE;   // masks are not exchanged
    for (int l = c->dmask_levels + 1; l <= (int)level; l++) {   // allocations outside the timed region
        const uint64_t n = c->lv[l].n;
        CKS(dalloc(c, (void**)&c->dmask[l], (n ? n : 1) * 64));
        CKS(cudaMemsetAsync(c->dmask[l], 0, (n ? n : 1) * 64, c->stream));
    }
    timer_begin(c, c->t_density);
    for (int l = c->dmask_levels + 1; l <= (int)level; l++) {
        CKS(launch_density_down(c, l));
        c->dmask_levels = l;
    }
    if (occ || axis) CKS(launch_density_stats(c, (int)level, occ, axis));
    if (masks && c->lv[level].n)
        CKS(cudaMemcpyAsync(masks, c->dmask[level], c->lv[level].n * 64, cudaMemcpyDefault, c->stream));
    timer_end(c, c->t_density);
    return VOX_OK;
}

vox_status vox_encode_level(vox_ctx* c, uint32_t level, uint8_t* sggx6, uint8_t* cl6, uint8_t* flags) {
    VOX_RANGE("vox_encode_level");
    if (!c || !sggx6) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    timer_begin(c, c->t_encode);
    CKS(launch_encode(c, c->lv[level], level == 0, sggx6, cl6, flags));
    timer_end(c, c->t_encode);
    c->st.launches++;
    return VOX_OK;
}

vox_status vox_copy_level(vox_ctx* c, uint32_t level, uint64_t* key, float* mass, float* m6, uint8_t* ncl, float* cl) {
    VOX_RANGE("vox_copy_level");
    if (!c) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    const Level& L = c->lv[level];
    const uint64_t n = L.n;
    const uint32_t K = c->K;
    if (n == 0) return VOX_OK;
    if (mass || m6 || (level > 0 && cl)) {
        vox_status s = ensure_f32(c, (int)level);
        if (s != VOX_OK) return s;
    }
    if (key) CKS(cudaMemcpyAsync(key, L.key, n * 8, cudaMemcpyDefault, c->stream));
    if (mass) CKS(cudaMemcpyAsync(mass, L.mass, n * 4, cudaMemcpyDefault, c->stream));
    if (m6) CKS(cudaMemcpyAsync(m6, L.m6, n * 24, cudaMemcpyDefault, c->stream));
    if (level > 0) {
        if (ncl) CKS(cudaMemcpyAsync(ncl, L.ncl, n, cudaMemcpyDefault, c->stream));
        if (cl) CKS(cudaMemcpyAsync(cl, L.cl, n * K * 28, cudaMemcpyDefault, c->stream));
    } else if (ncl || cl) {
        uint8_t* dn = nullptr;
        float* dc = nullptr;
        if (ncl) CKS(dalloc(c, (void**)&dn, n));
        if (cl) CKS(dalloc(c, (void**)&dc, n * K * 28));
        uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 32);
        k_leaf_lobes<<<(unsigned)blocks, 256, 0, c->stream>>>(n, L.acc, (int)K, dn, dc);
        c->st.launches++;
        if (ncl) CKS(cudaMemcpyAsync(ncl, dn, n, cudaMemcpyDefault, c->stream));
        if (cl) CKS(cudaMemcpyAsync(cl, dc, n * K * 28, cudaMemcpyDefault, c->stream));
        dfree(c, dn);
        dfree(c, dc);
    }
    CKS(ssync(c));
    return VOX_OK;
}

vox_status vox_copy_level_async(vox_ctx* c, uint32_t level, uint64_t* key, float* mass, float* m6, uint8_t* ncl,
                                float* cl, void* stream) {
    VOX_RANGE("vox_copy_level_async");
    if (!c) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    if (level == 0 && (ncl || cl)) return VOX_ERR_INVALID_ARG;
    const Level& L = c->lv[level];
    const uint64_t n = L.n;
    if (n == 0) return VOX_OK;
    cudaStream_t s = (cudaStream_t)stream;
    // key / mass / m6 are final once the level's prep ran (event recorded by the build), the
    // lobes once everything enqueued so far has run
    if (c->ev_level_ok[level]) CKS(cudaStreamWaitEvent(s, c->ev_level[level], 0));
    else if (key || mass || m6) {
        cudaEvent_t e0;
        CKS(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
        CKS(cudaEventRecord(e0, c->stream));
        CKS(cudaStreamWaitEvent(s, e0, 0));
        CKS(cudaEventDestroy(e0));
    }
    // the fp32 views are formed from the accumulators on `s` into stream-ordered scratch from
    // the device pool (cudaMallocAsync / cudaFreeAsync on `s`), unless the level already holds
    // them, so the build on the ctx stream is not delayed
    const bool have = L.f32;
    if (key) CKS(cudaMemcpyAsync(key, L.key, n * 8, cudaMemcpyDefault, s));
    if (have && (mass || m6)) {   // views formed by an earlier read: ordered after it
        cudaEvent_t e1;
        CKS(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        CKS(cudaEventRecord(e1, c->stream));
        CKS(cudaStreamWaitEvent(s, e1, 0));
        CKS(cudaEventDestroy(e1));
    }
    if (mass || m6) {
        float *tm = have ? L.mass : nullptr, *t6 = have ? L.m6 : nullptr;
        if (!have) {
            if (mass) CKS(cudaMallocAsync((void**)&tm, n * 4, s));
            if (m6) CKS(cudaMallocAsync((void**)&t6, n * 24, s));
            CKS(launch_finalize(c, s, n, L.acc, nullptr, nullptr, mass ? tm : nullptr, m6 ? t6 : nullptr, nullptr));
        }
        if (mass) CKS(cudaMemcpyAsync(mass, tm, n * 4, cudaMemcpyDefault, s));
        if (m6) CKS(cudaMemcpyAsync(m6, t6, n * 24, cudaMemcpyDefault, s));
        if (!have) {
            if (tm) CKS(cudaFreeAsync(tm, s));
            if (t6) CKS(cudaFreeAsync(t6, s));
        }
    }
    cudaEvent_t ev;
    CKS(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CKS(cudaEventRecord(ev, c->stream));      // after everything that produced the level
    CKS(cudaStreamWaitEvent(s, ev, 0));
    CKS(cudaEventDestroy(ev));
    if (ncl) CKS(cudaMemcpyAsync(ncl, L.ncl, n, cudaMemcpyDefault, s));
    if (cl) {
        float* tc = have ? L.cl : nullptr;
        if (!have) {
            CKS(cudaMallocAsync((void**)&tc, n * c->K * 28, s));
            CKS(launch_finalize(c, s, n, nullptr, L.ncl, L.clacc, nullptr, nullptr, tc));
        }
        CKS(cudaMemcpyAsync(cl, tc, n * c->K * 28, cudaMemcpyDefault, s));
        if (!have) CKS(cudaFreeAsync(tc, s));
    }
    // the level's arrays are being read on `s` until here: free_level / import wait on it
    if (!c->ev_read[level]) CKS(cudaEventCreateWithFlags(&c->ev_read[level], cudaEventDisableTiming));
    CKS(cudaEventRecord(c->ev_read[level], s));
    c->ev_read_pending[level] = true;
    return VOX_OK;
}

vox_status vox_copy_level_acc(vox_ctx* c, uint32_t level, int64_t* acc) {
    VOX_RANGE("vox_copy_level_acc");
    if (!c || !acc) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    const Level& L = c->lv[level];
    if (L.n == 0) return VOX_OK;
    CKS(cudaMemcpyAsync(acc, L.acc, L.n * 56, cudaMemcpyDefault, c->stream));
    CKS(ssync(c));
    return VOX_OK;
}

vox_status vox_export_level(vox_ctx* c, uint32_t level, void* buf, uint64_t* bytes) {
    VOX_RANGE("vox_export_level");
    if (!c || !bytes) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->built) return VOX_ERR_LEVEL;
    const uint64_t need = c->lv[level].n * record_bytes(c->K);
    if (!buf) {
        *bytes = need;
        return VOX_OK;
    }
    if (*bytes < need) return VOX_ERR_COMM;
    CKS(launch_pack(c, (int)level, buf));
    *bytes = need;
    return VOX_OK;
}

vox_status vox_import_level(vox_ctx* c, uint32_t level, const void* buf, uint64_t bytes) {
    VOX_RANGE("vox_import_level");
    if (!c) return VOX_ERR_INVALID_ARG;
    if ((int)level > c->g.logN) return VOX_ERR_LEVEL;
    const uint64_t rb = record_bytes(c->K);
    if (bytes % rb != 0 || (bytes && !buf)) return VOX_ERR_COMM;
    vox_status s = ensure_dev(c);
    if (s != VOX_OK) return s;
    for (int l = (int)level + 1; l < VOX_MAX_LEVELS; l++) free_level(c, c->lv[l]);
    for (int l = (int)level; l < VOX_MAX_LEVELS; l++) c->ev_level_ok[l] = false;   // arrays replaced
    // sub-voxel masks of the replaced levels were sized for the old arrays: drop them (the
    // masks are per shard and are not exchanged, vox_density_level refuses gathered levels)
    for (int l = (int)level; l < VOX_MAX_LEVELS; l++)
        if (c->dmask[l]) {
            dfree(c, c->dmask[l]);
            c->dmask[l] = nullptr;
        }
    if (c->dmask_levels >= (int)level) c->dmask_levels = (int)level - 1;
    s = unpack_level(c, (int)level, buf, bytes / rb);
    if (s != VOX_OK) return s;
    c->imported_level = (int)level;
    c->built = (int)level;
    if (c->state == ST_CREATED) c->state = ST_VOXELIZED;
    return VOX_OK;
}

vox_status vox_theta_table(float* theta, float* coef) {
    if (!theta || !coef) return VOX_ERR_INVALID_ARG;
    float t[32][3], k[32][6];
    host_theta(t, k);
    std::memcpy(theta, t, sizeof(t));
    std::memcpy(coef, k, sizeof(k));
    return VOX_OK;
}

vox_status vox_hist_tables(uint32_t N, float* u, uint8_t* perm, uint32_t* gap) {
    if (N < 32 || N > 8160) return VOX_ERR_INVALID_ARG;
    std::vector<float> hu;
    std::vector<uint8_t> hp;
    std::vector<uint32_t> hg;
    host_hist_tables((int)N, hu, hp, hg);
    if (u) std::memcpy(u, hu.data(), hu.size() * sizeof(float));
    if (perm) std::memcpy(perm, hp.data(), hp.size());
    if (gap) std::memcpy(gap, hg.data(), hg.size() * sizeof(uint32_t));
    return VOX_OK;
}

vox_status vox_debug_flags(uint32_t* out) {
    if (!out) return VOX_ERR_INVALID_ARG;
    *out = debug_read_fiber() | debug_read_reduce() | debug_read_lod();
    return VOX_OK;
}

vox_status vox_stats_get(vox_ctx* c, vox_stats* out) {
    if (!c || !out) return VOX_ERR_INVALID_ARG;
    CKS(ssync(c));
    c->st.ms_bound = timer_flush(c, c->t_bound);
    c->st.ms_emit = timer_flush(c, c->t_emit);
    c->st.ms_sort = timer_flush(c, c->t_sort);
    c->st.ms_reduce = timer_flush(c, c->t_reduce);
    c->st.ms_merge = timer_flush(c, c->t_merge);
    c->st.ms_lod_scan = timer_flush(c, c->t_lodscan);
    c->st.ms_lod = timer_flush(c, c->t_lod);
    c->st.ms_total_vox = timer_flush(c, c->t_vox);
    c->st.ms_total_lod = timer_flush(c, c->t_lodall);
    c->st.ms_lod_prep = timer_flush(c, c->t_prep);
    c->st.ms_sggxh_quad = timer_flush(c, c->t_quad);
    c->st.ms_sggxh_half = timer_flush(c, c->t_half);
    c->st.ms_sggxh_warp = timer_flush(c, c->t_warp);
    c->st.ms_encode = timer_flush(c, c->t_encode);
    c->st.ms_density = timer_flush(c, c->t_density);
    if (c->d_lodwork) {
        unsigned long long w[3] = {0, 0, 0};
        CKS(readback(c, {{w, c->d_lodwork, 24}}));
        c->st.lod_sigma_evals = w[0];
        c->st.lod_dist_evals = w[1];
        c->st.lod_hard_parents = w[2];
    }
    *out = c->st;
    return VOX_OK;
}

vox_status vox_stats_reset(vox_ctx* c) {
    if (!c) return VOX_ERR_INVALID_ARG;
    vox_stats tmp;
    vox_stats_get(c, &tmp);
    for (StageTimer* t : {&c->t_bound, &c->t_emit, &c->t_sort, &c->t_reduce, &c->t_merge, &c->t_lodscan, &c->t_lod,
                          &c->t_vox, &c->t_lodall, &c->t_prep, &c->t_quad, &c->t_half, &c->t_warp, &c->t_encode, &c->t_density})
        t->ms = 0.0;
    c->st.launches = 0;
    c->st.host_ms_alloc = c->st.host_ms_sync = 0;
    c->st.lod_sigma_evals = c->st.lod_dist_evals = c->st.lod_hard_parents = 0;
    if (c->d_lodwork) CKS(cudaMemsetAsync(c->d_lodwork, 0, 32, c->stream));
    return VOX_OK;
}

vox_status vox_trim(vox_ctx* c) {
    VOX_RANGE("vox_trim");
    if (!c) return VOX_ERR_INVALID_ARG;
    CKS(ssync(c));
    vox_trim_stream(c->stream);
    CKS(ssync(c));
    return VOX_OK;
}

vox_status vox_sync(vox_ctx* c) {
    VOX_RANGE("vox_sync");
    if (!c) return VOX_ERR_INVALID_ARG;
    CKS(ssync(c));
    return VOX_OK;
}

void vox_destroy(vox_ctx* c) {
    VOX_RANGE("vox_destroy");
    if (!c) return;
    ssync(c);
    release_mapped(c);
    density_reset(c);
    for (int l = 0; l < VOX_MAX_LEVELS; l++) free_level(c, c->lv[l]);
    for (int l = 0; l < VOX_MAX_LEVELS; l++) {
        if (c->ev_level[l]) cudaEventDestroy(c->ev_level[l]);
        if (c->ev_read[l]) cudaEventDestroy(c->ev_read[l]);
    }
    for (StageTimer* t : {&c->t_bound, &c->t_emit, &c->t_sort, &c->t_reduce, &c->t_merge, &c->t_lodscan, &c->t_lod,
                          &c->t_vox, &c->t_lodall, &c->t_prep, &c->t_quad, &c->t_half, &c->t_warp, &c->t_encode, &c->t_density}) {
        timer_flush(c, *t);
        if (t->open) cudaEventDestroy(t->open);
    }
    {
        std::lock_guard<std::mutex> lk(g_ev_mu);
        for (cudaEvent_t e : c->ev_pool) g_ev_pool[c->dev].push_back(e);
    }
    c->ev_pool.clear();
    if (c->d_lodwork) cudaFreeAsync(c->d_lodwork, c->stream);
    if (c->d_flags) cudaFreeAsync(c->d_flags, c->stream);
    if (c->d_counter) cudaFreeAsync(c->d_counter, c->stream);
    ssync(c);
    delete c;
}

}  // extern "C"
