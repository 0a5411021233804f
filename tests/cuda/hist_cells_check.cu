// Checks hist_cell_fast against hist_cell_pinned (paper_2604_13191_b200/csrc/hist_cells.cuh):
// whenever the fast path decides a cell, it is the pinned one. Inputs: random vectors over a
// wide range of magnitudes, and vectors built so that one normalised component sits within
// +-64 ulps of each cell boundary (d = -0.6, -0.2, 0.2, 0.6) -- where a wrong shortcut would
// show. Prints "mismatches M fast F total T" and exits non-zero on a mismatch.
#include <cstdio>
#include <cstdint>
#include "../../paper_2604_13191_b200/csrc/hist_cells.cuh"

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ float unit(uint32_t h) { return (float)(h >> 8) * (1.0f / 16777216.0f); }  // [0, 1)

__global__ void k_check(unsigned long long* cnt, uint32_t nrand, uint32_t nnear) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    unsigned long long bad = 0, fast = 0, tot = 0;
    const float bnd[4] = {-0.6f, -0.2f, 0.2f, 0.6f};
    for (uint32_t s = tid; s < nrand + nnear; s += stride) {
        float v[3];
        const uint32_t h0 = mix(2u * s + 1u), h1 = mix(h0 ^ 0x9e3779b9u), h2 = mix(h1 ^ 0x85ebca6bu), h3 = mix(h2 ^ 0xc2b2ae35u);
        if (s < nrand) {   // random direction, magnitude 2^[-40, 40)
            const float sc = exp2f(-40.0f + 80.0f * unit(h3));
            v[0] = (2.0f * unit(h0) - 1.0f) * sc;
            v[1] = (2.0f * unit(h1) - 1.0f) * sc;
            v[2] = (2.0f * unit(h2) - 1.0f) * sc;
        } else {           // component c at boundary b, perturbed by k ulps
            const uint32_t q = s - nrand;
            const int c = (int)(q % 3u), bi = (int)((q / 3u) % 4u), k = (int)((q / 12u) % 129u) - 64;
            const float b = bnd[bi];
            const float o1 = 2.0f * unit(h0) - 1.0f, o2 = 2.0f * unit(h1) - 1.0f;
            const float rest = sqrtf(o1 * o1 + o2 * o2) + 1e-3f;
            float vc = b * rest / sqrtf(1.0f - b * b);
            vc = __int_as_float(__float_as_int(vc) + k);
            v[c] = vc;
            v[(c + 1) % 3] = o1 + 1e-3f;
            v[(c + 2) % 3] = o2;
        }
        const float n2 = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
        if (!(n2 > 0.0f)) continue;
        tot++;
        const int f = vox::hist_cell_fast(v[0], v[1], v[2], n2);
        if (f >= 0) {
            fast++;
            bad += f != vox::hist_cell_pinned(v[0], v[1], v[2], n2);
        }
    }
    atomicAdd(&cnt[0], bad);
    atomicAdd(&cnt[1], fast);
    atomicAdd(&cnt[2], tot);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 24);
    cudaMemset(d, 0, 24);
    k_check<<<148 * 8, 256>>>(d, 1u << 27, 1u << 24);
    unsigned long long h[3] = {~0ull, 0, 0};
    if (cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
    printf("mismatches %llu fast %llu total %llu\n", h[0], h[1], h[2]);
    return h[0] == 0 && h[1] > 0 ? 0 : 1;
}
