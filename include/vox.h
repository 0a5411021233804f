/*
 * vox.h -- C ABI of the B200-native sparse voxelizer + SGGX-H LoD builder.
 *
 * Method: "Fast Voxelization and Level of Detail for Microgeometry Rendering"
 * (arXiv 2604.13191). P:n = line n of the paper's LaTeX; docs/PREDICATES.md
 * (§n) pins every operation; DESIGN.md lists the readings (Dn) of the paper.
 *
 * Conventions (all entry points):
 *   - C linkage, no exceptions cross the ABI; every call returns a vox_status.
 *   - Device pointers are CUDA device (or managed) memory, fp32 contiguous, 4-byte
 *     aligned (16-byte alignment is faster, not required). They are caller-owned and must
 *     stay valid until the call's work completes on the ctx stream (vox_sync).
 *   - Every call is ordered on the ctx stream (vox_options.stream, a cudaStream_t; NULL =
 *     the legacy default stream). The only internal host synchronisations are the small
 *     device->host reads that size allocations (documented per call).
 *   - Outputs are owned by the ctx. Views returned by vox_read_level stay valid until the
 *     next mutating call on the ctx or vox_destroy.
 *   - A ctx is not thread-safe; distinct ctxs are independent.
 *   - Results are bit-identical for identical (grid_res, bbox, options, multiset of
 *     primitives), independent of primitive order, batch splits, run and GPU count
 *     (exact integer accumulation, PREDICATES §8).
 */
#ifndef VOX_H
#define VOX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vox_ctx vox_ctx;

typedef enum {
    VOX_OK = 0,
    VOX_ERR_INVALID_ARG = 1,     /* bad argument, NaN/Inf input, negative radius, zero dir */
    VOX_ERR_DEGENERATE_BBOX = 2, /* non-finite bbox or b_max <= b_min on an axis */
    VOX_ERR_STATE = 3,           /* call not allowed in the ctx's current state */
    VOX_ERR_OOM = 4,             /* device allocation failed */
    VOX_ERR_CAPACITY = 5,        /* estimated bytes exceed vox_options.max_bytes */
    VOX_ERR_CUDA = 6,            /* a CUDA runtime error (see vox_last_error) */
    VOX_ERR_LEVEL = 7,           /* level out of range or not built yet */
    VOX_ERR_COMM = 8             /* export/import buffer malformed or too small */
} vox_status;

/* Zero-initialised = defaults. */
typedef struct {
    void* stream;          /* cudaStream_t for every call (NULL = default stream) */
    int rank;              /* Morton-range shard of this ctx, 0..world-1 (default 0) */
    int world;             /* number of shards (default 1 = unsharded) */
    int top_depth;         /* T: sharding/binning by Morton prefixes of 3T bits; 0 = min(4, log2 N) */
    uint32_t k;            /* max SGGX lobes kept per voxel, 1..8 (default 3) */
    uint32_t n_slices;     /* slice directions of the SGGX-H distance: 32 only (default 32) */
    uint64_t max_bytes;    /* cap on scratch+output device bytes per call (0 = no cap) */
    int profile;           /* 1 = record per-stage CUDA events (vox_stats times) */
    int distance_mode;     /* SGGX-H distance: 0 = sigma (PREDICATES §9, default), 1 = the paper's
                            * histogram distance (§10: N samples per SGGX, 5x5x5 bins, sliced W1;
                            * P:383-389) */
    uint32_t hist_samples; /* N of distance_mode 1, 32..8160 (0 = 5000) */
    uint64_t part_candidates; /* candidate voxels per Morton part of one voxelize call
                               * (0 = 3*2^30, also the maximum): a call with more candidates
                               * runs part by part over this rank's top-cell range, which
                               * bounds its pair scratch (16 B per candidate); the result is
                               * identical */
} vox_options;

/* Level view. Level 0 (leaves): ncl and cl are NULL; a leaf holds exactly one lobe
 * (mass, M) iff mass > 0. */
typedef struct {
    uint64_t n;            /* voxels in the level (this rank's part for local levels) */
    const uint64_t* key;   /* [n] Morton keys of the level (key >> 3l of leaf keys), ascending */
    const float* mass;     /* [n] density mass (PREDICATES §5, §7; D9) */
    const float* m6;       /* [n][6] second moment M: xx, yy, zz, xy, xz, yz (SGGX S = M / mass) */
    const uint8_t* ncl;    /* [n] number of SGGX-H lobes kept (<= k), or NULL for level 0 */
    const float* cl;       /* [n][k][7] lobes (w, M6); slots >= ncl are zero; NULL for level 0 */
    const int64_t* acc;    /* [n][7] exact fixed-point accumulators (quantum 2^-32) */
} vox_level_view;

typedef struct {
    uint64_t segments;     /* primitives read by the last voxelize call */
    uint64_t candidates;   /* in-grid, in-shard candidate voxels (upper bound on pairs) */
    uint64_t pairs;        /* (key, contribution) pairs emitted by the last call */
    uint64_t voxels;       /* leaf voxels after the last call */
    uint32_t top_depth;    /* T in use */
    uint64_t cell_lo, cell_hi; /* this rank's top-cell range [lo, hi) */
    /* accumulated device milliseconds per stage since the last vox_stats_reset (profile=1) */
    double ms_bound, ms_emit, ms_sort, ms_reduce, ms_merge, ms_lod_scan, ms_lod, ms_total_vox, ms_total_lod;
    double ms_lod_prep, ms_sggxh_quad, ms_sggxh_half, ms_sggxh_warp;   /* parts of ms_lod: sums, SGGX-H n<=8, 9..16, >16 (hist mode: all in warp) */
    uint64_t launches;     /* kernels launched by the library since the last reset */
    /* SGGX-H algorithmic work since the last reset (profile=1): lobe sigma evaluations
     * (32 slices each), pair distance evaluations (32 slices each), parents with n > k */
    uint64_t lod_sigma_evals, lod_dist_evals, lod_hard_parents;
    double host_ms_alloc, host_ms_sync;   /* host time in stream-ordered allocation / stream syncs */
    double ms_encode;      /* vox_encode_level device time (profile=1) */
    double ms_density;     /* vox_density_* device time (profile=1) */
} vox_stats;

/* Create a ctx for an N^3 grid over the cubic extent of bbox (D3).
 * grid_res: power of two in [2, 8192] (D27) else VOX_ERR_INVALID_ARG.
 * bbox: host float[6] = min xyz, max xyz; must be finite with max > min per axis
 * (else VOX_ERR_DEGENERATE_BBOX). opt: host pointer or NULL (defaults). No device
 * allocation happens here. The first call that touches the device configures the device's
 * default memory pool process-wide: release threshold unlimited (freed stream-ordered memory
 * stays mapped for the next call) and no internal cross-stream dependencies (memory freed on
 * one stream is not handed to another by making it wait; completed frees are still reused). */
vox_status vox_create(vox_ctx** out, uint32_t grid_res, const float bbox[6], const vox_options* opt);

/* Voxelize S fiber segments (capsules; PREDICATES §3-§5, north star).
 * segments: device float[S][2][3] world-space endpoints; radii: device float[S] (>= 0).
 * Accumulates into the leaf level (D19). S = 0 is a no-op VOX_OK (D26).
 * NaN/Inf coordinates, negative radii or a segment with > 2^24 candidate voxels ->
 * VOX_ERR_INVALID_ARG (detected on the device; the leaf level is unchanged).
 * Host syncs: 2 small reads (per-top-cell candidate counts; emitted pair count). */
vox_status vox_voxelize_fibers(vox_ctx* ctx, const float* segments, const float* radii, uint64_t S);

/* Voxelize T triangles (PREDICATES §6-§7). tris: device float[T][3][3] world
 * vertices (soup); dirs: device float[T][3] per-triangle direction (tangent mode,
 * P:183) or NULL for face normals. A zero-norm dir -> VOX_ERR_INVALID_ARG. */
vox_status vox_voxelize_triangles(vox_ctx* ctx, const float* tris, const float* dirs, uint64_t T);

/* Same as the two calls above with HOST input pointers (pinned memory is fastest): the
 * host->device copies run on the ctx stream inside the call. */
vox_status vox_voxelize_fibers_host(vox_ctx* ctx, const float* segments, const float* radii, uint64_t S);
vox_status vox_voxelize_triangles_host(vox_ctx* ctx, const float* tris, const float* dirs, uint64_t T);

/* Build levels 1..levels of the 2x2x2 Morton pyramid with SGGX-H per parent
 * (PREDICATES §9). levels <= log2(grid_res) else VOX_ERR_LEVEL. Levels already
 * built are kept; voxelize_* afterwards returns VOX_ERR_STATE. Sharded ctx (world > 1):
 * builds at most up to level log2(N) - T until vox_import_level(log2(N) - T) has been
 * called (query vox_built_levels). Host syncs: one 8-byte read per level. */
vox_status vox_build_lod(vox_ctx* ctx, uint32_t levels);

/* Highest level available for reading (0 after create). */
vox_status vox_built_levels(vox_ctx* ctx, uint32_t* out);

/* Number of voxels of a built level (no device work, no sync). level > built ->
 * VOX_ERR_LEVEL; out NULL -> VOX_ERR_INVALID_ARG. */
vox_status vox_level_size(vox_ctx* ctx, uint32_t level, uint64_t* out);

/* Borrowed view of a level (see vox_level_view). level > built -> VOX_ERR_LEVEL. The build
 * keeps only keys, the exact accumulators and lobe accumulators; the first read of a level
 * allocates its fp32 views (mass, m6, cl: one rounding of each fixed-point sum, PREDICATES
 * §8) and fills them on the ctx stream, so the view is valid once the stream reaches that
 * point (vox_sync). Allocation failure -> VOX_ERR_OOM. */
vox_status vox_read_level(vox_ctx* ctx, uint32_t level, vox_level_view* out);

/* Copy a level into caller-owned buffers (device or host; any pointer may be NULL):
 * key [n], mass [n], m6 [n][6], ncl [n], cl [n][k][7]. Level 0 copies ncl = (mass > 0)
 * and cl = (mass, M) in slot 0. Forms the level's fp32 views first if needed (as
 * vox_read_level). Synchronises the ctx stream. */
vox_status vox_copy_level(vox_ctx* ctx, uint32_t level, uint64_t* key, float* mass, float* m6,
                          uint8_t* ncl, float* cl);

/* The paper's own sampling front end (PREDICATES §12; §3.2):
 * primitives become samples, each sample adds (mass, mass * d d^T) to the voxel containing it
 * (half-open cells, samples outside [0,N)^3 dropped); the pairs go through the same binned
 * reduce as the exact path and calls accumulate with every other voxelize call (D19).
 *   vox_sample_splines: Catmull-Rom pieces, ctrl dev f32 [S][4][3] (P0..P3 world; the piece
 *     runs P1 -> P2), radii dev f32 [S]; n samples per piece at t = (s + 1/2)/n, each
 *     with mass pi r^2 |P2 - P1| / n (grid units) and the curve's unit tangent.
 *     n in 1..65536 and S * n < 2^32, else VOX_ERR_INVALID_ARG.
 *   vox_sample_triangles: tris dev f32 [T][3][3], dirs dev f32 [T][3] or NULL (face normals);
 *     round(budget * A / A_max) samples per triangle (>= 1 if A > 0; A_max over the call,
 *     P:228) placed by Heitz's low-distortion square -> triangle map, each with mass
 *     A / n_t. budget in 1..65536.
 * Non-finite input, negative radius or zero dirs -> VOX_ERR_INVALID_ARG at the call's sync. */
vox_status vox_sample_splines(vox_ctx* ctx, const float* ctrl, const float* radii, uint64_t S, uint32_t n);
vox_status vox_sample_triangles(vox_ctx* ctx, const float* tris, const float* dirs, uint64_t T, uint32_t budget);

/* Sub-voxel occupancy and axis-projected densities (PREDICATES §13; P:282-291, P:347-349,
 * S:266-271). Res_3 = 8: sub-voxel (a,b,c) of voxel (i,j,k) is hit iff
 * the key predicate (§4 fibers / §6 triangles) holds for fine voxel (8i+a, 8j+b, 8k+c) of the
 * 8N grid. vox_density_fibers / _triangles OR the hits of the given primitives (device
 * arrays as in vox_voxelize_*) into per-voxel 512-bit masks of level 0; call them after the
 * last voxelize call (a voxelize call resets the masks), once per primitive batch.
 * Before any voxelize call -> VOX_ERR_STATE. Inputs are assumed validated by voxelize.
 * vox_density_level(level): occ [n] = hits / 512, axis [n][3] = projected coverage onto the
 * YZ, XZ, XY planes / 64, masks [n][8] (word z, bit x + 8 y; NULL = skipped) into caller
 * device buffers; level > 0 masks are the 2x2x2 OR-downsampling of level - 1 (built lazily).
 * No masks yet -> VOX_ERR_STATE; level > built -> VOX_ERR_LEVEL; sharded ctx: levels above
 * log2(N) - T -> VOX_ERR_STATE (masks are not exchanged). */
vox_status vox_density_fibers(vox_ctx* ctx, const float* segments, const float* radii, uint64_t S);
vox_status vox_density_triangles(vox_ctx* ctx, const float* tris, uint64_t T);
vox_status vox_density_level(vox_ctx* ctx, uint32_t level, float* occ, float* axis, uint64_t* masks);

/* SGGX finalisation and the 6-byte compact form (PREDICATES §11; Eq. compact-sggx P:354-362,
 * SPEC S:47) of every record of a level, into
 * caller-owned DEVICE buffers (stream-ordered on the ctx stream, no sync):
 *   sggx6 [n][6]    the voxel's aggregate (mass, M): sigma_x, sigma_y, sigma_z bytes
 *                   (round(sigma*255)), r_xy, r_xz, r_yz bytes (round((r+1)*127.5)), after
 *                   the degenerate jitter (lambda_min < 1e-4 lambda_max) and normalisation to
 *                   maximum projected area 1; a record with w = 0 is (0,0,0,128,128,128);
 *   cl6   [n][k][6] the voxel's SGGX-H lobes, slots >= ncl as for w = 0 (NULL: skipped);
 *                   at level 0 slot 0 is the voxel itself;
 *   flags [n]       bit 0: aggregate jittered, bit 1+q: lobe q jittered (NULL: skipped).
 * level > built -> VOX_ERR_LEVEL; sggx6 NULL -> VOX_ERR_INVALID_ARG. */
vox_status vox_encode_level(vox_ctx* ctx, uint32_t level, uint8_t* sggx6, uint8_t* cl6, uint8_t* flags);

/* Like vox_copy_level but asynchronous on the caller's `stream` (a cudaStream_t, NULL = the
 * legacy default stream) and without synchronising: key / mass / m6 are ordered after the
 * level's prep (they are final there; an event recorded by the build), ncl / cl after all
 * work enqueued on the ctx stream so far (an event), so the D2H of level l overlaps the
 * clustering of level l and the build of levels > l. Building further levels does not touch
 * lower levels; the caller synchronises `stream` before reading the buffers or destroying
 * the ctx. The fp32 values are formed from the accumulators by a small kernel on `stream`
 * into stream-ordered scratch from the device pool (allocated and freed on `stream`) before
 * each D2H; a level whose views an earlier read formed is copied from them, after that read.
 * Those kernels share the SMs with the build still running on the ctx stream: give `stream`
 * a high priority (cudaStreamCreateWithPriority) so they are scheduled ahead of the build's
 * blocks and the copy engine is not left idle behind them (bench.py does).
 * Level 0 supports key / mass / m6 only (ncl or cl non-NULL -> VOX_ERR_INVALID_ARG). */
vox_status vox_copy_level_async(vox_ctx* ctx, uint32_t level, uint64_t* key, float* mass, float* m6,
                                uint8_t* ncl, float* cl, void* stream);

/* Debug builds (-DVOX_DEBUG): OR of the bounds-check bits that fired since the last call
 * (bit 0 emit survivor FIFO, 1 bin rank, 2 bin slot, 3 warp-kernel lobe count, 4 quad lobe
 * count, 5 half lobe count, 7 level-1 staged rows), cleared by the read; release builds
 * always return 0. Synchronous (reads device memory). */
vox_status vox_debug_flags(uint32_t* out);

/* Copy a level's exact accumulators acc [n][7] (int64, quantum 2^-32; device or host). */
vox_status vox_copy_level_acc(vox_ctx* ctx, uint32_t level, int64_t* acc);

/* Multi-GPU (Morton-range shards). A level's records are fixed-size:
 * key u64, acc i64[7], ncl u64 (low byte), lobe accumulators i64[k][7]  ->  72 + 56k bytes.
 * export: dev_buf == NULL -> *bytes = required size; else writes the records of this rank
 * (device memory, *bytes must be >= required; on return *bytes = bytes written).
 * import: replaces `level` with the concatenation of all ranks' records in rank order
 * (ascending keys), which must be level log2(N) - T; afterwards vox_build_lod can build
 * the top levels redundantly on every rank. Bad sizes or unsorted keys -> VOX_ERR_COMM. */
vox_status vox_export_level(vox_ctx* ctx, uint32_t level, void* dev_buf, uint64_t* bytes);
vox_status vox_import_level(vox_ctx* ctx, uint32_t level, const void* dev_buf, uint64_t bytes);

/* Deterministic work-balanced partition of 8^T top cells over `world` ranks (host only,
 * no GPU needed): bounds[r] = first cell of rank r, bounds[world] = ncells; rank r owns
 * [bounds[r], bounds[r+1]). weights[c] = candidate voxels in cell c. The first voxelize
 * call of a sharded ctx computes this from its candidate counts and freezes it. */
vox_status vox_plan_shards(const uint64_t* weights, uint64_t ncells, int world, uint64_t* bounds);

/* Host copy of the SGGX-H slice table (PREDICATES §9): theta [32][3], coef [32][6]. */
vox_status vox_theta_table(float* theta, float* coef);

/* Host copy of the histogram-distance tables (PREDICATES §10) for N samples (32..8160):
 * u [3][N] whole-sphere sample table (SoA x, y, z), perm [124][32] the first 124 sorted
 * cells of each slice (transposed: perm[r*32 + k]), gap [124][32] the fixed-point gaps.
 * Any pointer may be NULL (not written). VOX_ERR_INVALID_ARG for N out of range. */
vox_status vox_hist_tables(uint32_t N, float* u, uint8_t* perm, uint32_t* gap);

vox_status vox_stats_get(vox_ctx* ctx, vox_stats* out);   /* synchronises the stream */
vox_status vox_stats_reset(vox_ctx* ctx);
/* Release the library's cached device blocks of the ctx stream (freed scratch and levels of
 * destroyed ctxs are kept for reuse by later calls on the same stream). */
vox_status vox_trim(vox_ctx* ctx);
vox_status vox_sync(vox_ctx* ctx);
const char* vox_status_str(vox_status s);
const char* vox_last_error(vox_ctx* ctx);
void vox_destroy(vox_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* VOX_H */
