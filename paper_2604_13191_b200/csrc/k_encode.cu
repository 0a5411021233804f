// SGGX finalisation and the 6-byte compact form (docs/PREDICATES.md §11; SURVEY §8(f) NEXT-3;
// Eq. compact-sggx): per record (a voxel's aggregate
// or one lobe) S = M / w, eigenvalues by the pinned cyclic Jacobi, the degenerate jitter in
// moment form, normalisation to maximum projected area 1, then sigma / r bytes.
//
// One thread per voxel (its aggregate and its K lobes); the block's byte outputs are staged in
// shared memory and written back as coalesced 32-bit words. ALU-bound: the pinned Jacobi is
// ~18 rotations with correctly rounded divisions and square roots per record.
#include "vox_internal.cuh"

namespace vox {

constexpr int ENC_THREADS = 256;

__device__ __forceinline__ void jacobi3(const float S[6], float lam[3]) {
    float a00 = S[0], a11 = S[1], a22 = S[2], a01 = S[3], a02 = S[4], a12 = S[5];
    // one rotation on (p, q) with r the third index; written out per pair so that every
    // matrix entry stays in a register
    auto rot = [](float& app, float& aqq, float& apq, float& arp, float& arq) -> int {
        // negligible off-diagonal (relative 2^-24 of the diagonal): no rotation
        if (!(fabsf(apq) * 16777216.0f > fabsf(app) + fabsf(aqq))) return 0;
        const float th = (aqq - app) / (2.0f * apq);
        float t = 1.0f / (fabsf(th) + sqrtf(th * th + 1.0f));
        if (th < 0.0f) t = -t;
        const float c = 1.0f / sqrtf(t * t + 1.0f);
        const float sn = t * c;
        app = app - t * apq;
        aqq = aqq + t * apq;
        apq = 0.0f;
        const float rp = arp, rq = arq;
        arp = c * rp - sn * rq;
        arq = sn * rp + c * rq;
        return 1;
    };
    for (int sweep = 0; sweep < 6; sweep++) {
        int rotated = rot(a00, a11, a01, a02, a12);   // (0,1), r = 2: a_r0 = a02, a_r1 = a12
        rotated |= rot(a00, a22, a02, a01, a12);      // (0,2), r = 1: a_r0 = a01, a_r2 = a12
        rotated |= rot(a11, a22, a12, a01, a02);      // (1,2), r = 0: a_r1 = a01, a_r2 = a02
        if (!rotated) break;                          // a sweep without rotation: converged
    }
    lam[0] = a00;
    lam[1] = a11;
    lam[2] = a22;
}

__device__ __forceinline__ uint8_t byte_sigma(float x) {
    const int b = (int)floorf(x * 255.0f + 0.5f);
    return (uint8_t)(b > 255 ? 255 : (b < 0 ? 0 : b));
}
__device__ __forceinline__ uint8_t byte_r(float r) {
    const int b = (int)floorf((r + 1.0f) * 127.5f + 0.5f);
    return (uint8_t)(b > 255 ? 255 : (b < 0 ? 0 : b));
}
__device__ __forceinline__ float corr(float sxy, float sxx, float syy) {
    const float p = sxx * syy;
    const float r = p > 0.0f ? sxy / sqrtf(p) : 0.0f;
    return r > 1.0f ? 1.0f : (r < -1.0f ? -1.0f : r);
}

// one record -> 6 bytes at out; returns 1 iff jittered
__device__ int encode_rec(const long long* __restrict__ acc, uint8_t* out) {
    out[0] = out[1] = out[2] = 0;
    out[3] = out[4] = out[5] = 128;
    const long long aw = acc[0];
    if (aw == 0) return 0;
    const float wf = deq32(aw);
    float S[6];
#pragma unroll
    for (int e = 0; e < 6; e++) S[e] = deq32(acc[1 + e]) / wf;
    const float tr = (S[0] + S[1]) + S[2];
    float lam[3];
    jacobi3(S, lam);
    float lmax = lam[0], lmin = lam[0];
#pragma unroll
    for (int a = 1; a < 3; a++) {
        if (lam[a] > lmax) lmax = lam[a];
        if (lam[a] < lmin) lmin = lam[a];
    }
    const int jit = lmin < 1e-4f * lmax;
    if (jit) {
        const float C1 = 0.9999f, C2 = (float)(1e-4 / 3.0);
#pragma unroll
        for (int e = 0; e < 6; e++) S[e] = e < 3 ? C1 * S[e] + C2 * tr : C1 * S[e];
        lmax = C1 * lmax + C2 * tr;
    }
    if (!(lmax > 0.0f)) return jit;
    const float inv = 1.0f / lmax;
    float Sn[6];
#pragma unroll
    for (int e = 0; e < 6; e++) Sn[e] = S[e] * inv;
    out[0] = byte_sigma(sqrtf(pmax(Sn[0], 0.0f)));
    out[1] = byte_sigma(sqrtf(pmax(Sn[1], 0.0f)));
    out[2] = byte_sigma(sqrtf(pmax(Sn[2], 0.0f)));
    out[3] = byte_r(corr(Sn[3], Sn[0], Sn[1]));
    out[4] = byte_r(corr(Sn[4], Sn[0], Sn[2]));
    out[5] = byte_r(corr(Sn[5], Sn[1], Sn[2]));
    return jit;
}

// copy `bytes` staged bytes to global dst (4-byte aligned when aligned4) cooperatively
__device__ __forceinline__ void flush_bytes(const uint8_t* src, uint8_t* dst, int bytes, bool aligned4) {
    if (aligned4) {
        const int w = bytes >> 2;
        for (int x = threadIdx.x; x < w; x += blockDim.x)
            reinterpret_cast<uint32_t*>(dst)[x] = reinterpret_cast<const uint32_t*>(src)[x];
        for (int x = (w << 2) + threadIdx.x; x < bytes; x += blockDim.x) dst[x] = src[x];
    } else {
        for (int x = threadIdx.x; x < bytes; x += blockDim.x) dst[x] = src[x];
    }
}

__global__ void __launch_bounds__(ENC_THREADS)
k_encode(uint64_t n, const long long* __restrict__ acc, const uint8_t* __restrict__ ncl,
         const long long* __restrict__ clacc, int K, uint8_t* __restrict__ out6, uint8_t* __restrict__ cl6,
         uint8_t* __restrict__ flags) {
    extern __shared__ __align__(16) uint8_t s_enc[];   // [256][6] aggregate | [256][K][6] lobes
    uint8_t* s_agg = s_enc;
    uint8_t* s_cl = s_enc + ENC_THREADS * 6;
    const bool a6 = (reinterpret_cast<uintptr_t>(out6) & 3) == 0;
    const bool ac = cl6 && (reinterpret_cast<uintptr_t>(cl6) & 3) == 0;
    for (uint64_t v0 = (uint64_t)blockIdx.x * ENC_THREADS; v0 < n; v0 += (uint64_t)gridDim.x * ENC_THREADS) {
        const uint64_t v = v0 + threadIdx.x;
        const int nb = (int)(n - v0 < (uint64_t)ENC_THREADS ? n - v0 : ENC_THREADS);
        if (v < n) {
            uint8_t f = (uint8_t)encode_rec(acc + 7 * v, s_agg + 6 * threadIdx.x);
            if (cl6) {
                uint8_t* o = s_cl + (size_t)threadIdx.x * K * 6;
                if (!clacc) {   // level 0: the voxel is its own single lobe
                    for (int e = 0; e < 6; e++) o[e] = s_agg[6 * threadIdx.x + e];
                    for (int q = 1; q < K; q++) {
                        o[6 * q] = o[6 * q + 1] = o[6 * q + 2] = 0;
                        o[6 * q + 3] = o[6 * q + 4] = o[6 * q + 5] = 128;
                    }
                    if (f) f |= 2;
                } else {
                    const int m = ncl[v];
                    for (int q = 0; q < K; q++) {
                        if (q < m) {
                            if (encode_rec(clacc + ((uint64_t)v * K + q) * 7, o + 6 * q)) f |= (uint8_t)(2u << q);
                        } else {
                            o[6 * q] = o[6 * q + 1] = o[6 * q + 2] = 0;
                            o[6 * q + 3] = o[6 * q + 4] = o[6 * q + 5] = 128;
                        }
                    }
                }
            }
            if (flags) flags[v] = f;
        }
        __syncthreads();
        flush_bytes(s_agg, out6 + 6 * v0, 6 * nb, a6 && ((6 * v0) & 3) == 0);
        if (cl6) flush_bytes(s_cl, cl6 + (size_t)6 * K * v0, 6 * K * nb, ac && ((6 * K * v0) & 3) == 0);
        __syncthreads();
    }
}

cudaError_t launch_encode(vox_ctx* c, const Level& L, int leaf, uint8_t* out6, uint8_t* cl6, uint8_t* flags) {
    if (L.n == 0) return cudaSuccess;
    const int K = (int)c->K;
    const size_t smem = (size_t)ENC_THREADS * 6 * (1 + K);
    uint64_t nb = (L.n + ENC_THREADS - 1) / ENC_THREADS;
    nb = std::min<uint64_t>(nb, 148ull * 8);
    k_encode<<<(unsigned)nb, ENC_THREADS, smem, c->stream>>>(L.n, L.acc, leaf ? nullptr : L.ncl,
                                                              leaf ? nullptr : L.clacc, K, out6, cl6, flags);
    return cudaGetLastError();
}

}  // namespace vox
