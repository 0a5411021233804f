// hist_cells.cuh -- the cell of a histogram sample (PREDICATES §10), the pinned sequence and
// the provably identical fast path used by k_hist.cu (tests/test_gpu_hist_cells.py checks
// them against each other, boundary neighbourhoods included). Product path.
#pragma once

namespace vox {

__device__ __forceinline__ int hist_bin1(float d) {
    const int b = (int)floorf((d + 1.0f) * 2.5f);
    return b < 0 ? 0 : (b > 4 ? 4 : b);
}

// The pinned cell of a sample (§10) without its IEEE square root and reciprocal, when that is
// provably the same cell: d'_c = fl(v_c * rsqrt.approx(n2)) differs from the pinned d_c =
// fl(v_c * fl(1 / fl(sqrt(n2)))) by < 4e-7 (|d| <= 1; rsqrt.approx's relative error is below
// 2^-22.9, the pinned sequence rounds three times), and x = fl(fl(d + 1) * 2.5) is monotone in
// d, so when x' is farther than 1e-5 from the cell boundaries 1..4 (boundaries 0 and 5 are
// clamped away) both land in the same cell. Returns -1 when a component is that close or n2
// is outside the normal range: the caller then takes the pinned sequence (hist_cell_pinned).
__device__ __forceinline__ int hist_axis_fast(float v, float rs, bool& near) {
    const float x = (v * rs + 1.0f) * 2.5f;
    const float k = rintf(x);
    near |= k >= 1.0f && k <= 4.0f && fabsf(x - k) <= 1e-5f;
    const int b = (int)floorf(x);
    return b < 0 ? 0 : (b > 4 ? 4 : b);
}
__device__ __forceinline__ int hist_cell_fast(float v0, float v1, float v2, float n2) {
    if (!(n2 >= 1.17549435e-38f && n2 <= 1.0e30f)) return -1;
    float rs;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(n2));
    bool near = false;
    const int b = hist_axis_fast(v0, rs, near) + 5 * hist_axis_fast(v1, rs, near) + 25 * hist_axis_fast(v2, rs, near);
    return near ? -1 : b;
}
__device__ __noinline__ int hist_cell_pinned(float v0, float v1, float v2, float n2) {
    const float r = sqrtf(n2);
    const float inv = 1.0f / r;
    return hist_bin1(v0 * inv) + 5 * hist_bin1(v1 * inv) + 25 * hist_bin1(v2 * inv);
}

}  // namespace vox
