// §13 sub-voxel occupancy and axis-projected densities (docs/PREDICATES.md §13; SURVEY §8(f)
// NEXT-2): level masks by 2x2x2 OR-downsampling of the children's
// 512-bit masks, then per voxel the occupancy popcount / 512 and the three projected
// coverages / 64. Level-0 masks come from k_fiber_density / k_tri_density.
#include "vox_internal.cuh"

namespace vox {

// thread per child voxel: its parent (binary search of key >> 3), its octant, the 4x4x4
// OR-downsample of its mask placed in the parent's 8x8x8 grid (atomicOr: siblings share words)
__global__ void k_density_down(const uint64_t* __restrict__ ckey, const unsigned long long* __restrict__ cm,
                               uint64_t nc, const uint64_t* __restrict__ pkey, uint64_t np,
                               unsigned long long* __restrict__ pm) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nc; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = ckey[v];
        const long long p = find_key(pkey, np, key >> 3);
        if (p < 0) continue;
        const int ox = (int)(key & 1), oy = (int)((key >> 1) & 1), oz = (int)((key >> 2) & 1);
#pragma unroll
        for (int zq = 0; zq < 4; zq++) {
            const unsigned long long t = cm[8 * v + 2 * zq] | cm[8 * v + 2 * zq + 1];
            if (!t) continue;
            unsigned long long out = 0;
#pragma unroll
            for (int bq = 0; bq < 4; bq++) {
                const unsigned rows = (unsigned)((t >> (16 * bq)) & 0xffffu);   // rows 2bq, 2bq+1
                const unsigned r = (rows | (rows >> 8)) & 0xffu;                  // OR of the two rows
#pragma unroll
                for (int aq = 0; aq < 4; aq++)
                    if ((r >> (2 * aq)) & 3u) out |= 1ull << ((4 * ox + aq) + 8 * (4 * oy + bq));
            }
            atomicOr(&pm[8 * p + 4 * oz + zq], out);
        }
    }
}

__global__ void k_density_stats(const unsigned long long* __restrict__ m, uint64_t n, float* __restrict__ occ,
                                float* __restrict__ axis) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long xy = 0, xz = 0, yz = 0;
        int hits = 0;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const unsigned long long w = m[8 * v + c];
            xy |= w;
            hits += __popcll(w);
            unsigned rowor = 0, colbits = 0;
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const unsigned row = (unsigned)((w >> (8 * b)) & 0xffu);
                rowor |= row;                          // OR over y: x bits of layer c
                colbits |= (row ? 1u : 0u) << b;       // OR over x: y bits of layer c
            }
            xz |= (unsigned long long)rowor << (8 * c);
            yz |= (unsigned long long)colbits << (8 * c);
        }
        if (occ) occ[v] = (float)hits / 512.0f;
        if (axis) {
            axis[3 * v + 0] = (float)__popcll(yz) / 64.0f;
            axis[3 * v + 1] = (float)__popcll(xz) / 64.0f;
            axis[3 * v + 2] = (float)__popcll(xy) / 64.0f;
        }
    }
}

cudaError_t launch_density_down(vox_ctx* c, int level) {
    const Level& C = c->lv[level - 1];
    const Level& P = c->lv[level];
    if (C.n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<uint64_t>((C.n + 255) / 256, 148ull * 32);
    k_density_down<<<grid, 256, 0, c->stream>>>(C.key, c->dmask[level - 1], C.n, P.key, P.n, c->dmask[level]);
    c->st.launches++;
    return cudaGetLastError();
}

cudaError_t launch_density_stats(vox_ctx* c, int level, float* occ, float* axis) {
    const uint64_t n = c->lv[level].n;
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 32);
    k_density_stats<<<grid, 256, 0, c->stream>>>(c->dmask[level], n, occ, axis);
    c->st.launches++;
    return cudaGetLastError();
}

}  // namespace vox
