// Tree keys of a point: the reference's quantisation (quadtree.py:177-185,
// f64 round-to-nearest, truncation) interleaved as a Morton code
// (quadtree.py:156-174) or keyed along the Hilbert curve (the engine's tree
// order).  Shared by k_morton (points.cu) and the fused key + histogram
// pass of the engine's sort (sort.cu).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace bh {

__device__ __forceinline__ uint32_t spread16(uint32_t x) {
    x &= 0xFFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

__device__ __forceinline__ uint64_t spread32(uint64_t m) {  // _spread_bits
    m &= 0x00000000FFFFFFFFull;
    m = (m | (m << 16)) & 0x0000FFFF0000FFFFull;
    m = (m | (m << 8)) & 0x00FF00FF00FF00FFull;
    m = (m | (m << 4)) & 0x0F0F0F0F0F0F0F0Full;
    m = (m | (m << 2)) & 0x3333333333333333ull;
    m = (m | (m << 1)) & 0x5555555555555555ull;
    return m;
}

// y - shift in the run precision (gradient_step's re-centering)
__device__ __forceinline__ float2 shifted(float2 p, const bh_bounds_t *b) {
    return make_float2(__fsub_rn(p.x, b->shift0), __fsub_rn(p.y, b->shift1));
}
__device__ __forceinline__ double2 shifted(double2 p, const bh_bounds_t *b) {
    return make_double2(__dsub_rn(p.x, b->shift0_f64),
                        __dsub_rn(p.y, b->shift1_f64));
}

// Hilbert index of the quantised cell (m0, m1), BITS/2 bits per dimension,
// the classic rotate-and-reflect walk from the top bit.  The top 2d bits of
// the index name the depth-d quadtree cell of the point (a bijection at
// every level), so the canonical tree over Hilbert keys has exactly the
// Morton tree's cells -- only siblings are ordered along the curve, which
// has no jumps between consecutive points.
template <int BITS, typename U>
__device__ __forceinline__ U hilbert_key(U x, U y) {
    // Branch-free form of the walk: the rotations and reflections applied so
    // far are a state (swap, comp) acting on the ORIGINAL bits of each level:
    // (xt, yt) = (swap ? (by, bx) : (bx, by)) ^ comp, digit = (3 xt) ^ yt,
    // and a level with yt == 0 toggles swap and, when xt == 1, comp.
    constexpr int H = BITS / 2;
    uint32_t swap = 0, comp = 0;
    U d = 0;
#pragma unroll
    for (int l = H - 1; l >= 0; l--) {
        const uint32_t bx = (uint32_t)(x >> l) & 1u, by = (uint32_t)(y >> l) & 1u;
        const uint32_t t = (bx ^ by) & swap;
        const uint32_t xt = bx ^ t ^ comp, yt = by ^ t ^ comp;
        d = (d << 2) | (U)(((xt << 1) | xt) ^ yt);
        const uint32_t z = yt ^ 1u;
        swap ^= z;
        comp ^= xt & z;
    }
    return d;
}

// The same walk four levels at a time: a 1024-entry table indexed by
// (state, 4 bits of x, 4 bits of y) gives the 8 key bits of those levels and
// the state after them (state = swap | comp << 1).  Built at compile time
// from the very recurrence of hilbert_key, so the keys are identical; the
// key kernel stages it in shared memory (4 lookups per 32-bit key instead
// of 16 dependent levels of ~12 operations).
struct HilbertLut {
    uint16_t v[1024];
};

constexpr HilbertLut make_hilbert_lut() {
    HilbertLut t{};
    for (uint32_t s = 0; s < 4; s++)
        for (uint32_t x = 0; x < 16; x++)
            for (uint32_t y = 0; y < 16; y++) {
                uint32_t swap = s & 1u, comp = s >> 1, d = 0;
                for (int l = 3; l >= 0; l--) {
                    const uint32_t bx = (x >> l) & 1u, by = (y >> l) & 1u;
                    const uint32_t u = (bx ^ by) & swap;
                    const uint32_t xt = bx ^ u ^ comp, yt = by ^ u ^ comp;
                    d = (d << 2) | (((xt << 1) | xt) ^ yt);
                    const uint32_t z = yt ^ 1u;
                    swap ^= z;
                    comp ^= xt & z;
                }
                t.v[(s << 8) | (x << 4) | y] =
                    (uint16_t)(((swap | (comp << 1)) << 8) | d);
            }
    return t;
}

__device__ const HilbertLut g_hilbert_lut = make_hilbert_lut();

// Stage the table in shared memory (every thread of the CTA calls this).
__device__ __forceinline__ void hilbert_lut_load(uint16_t *s_lut) {
    for (int i = threadIdx.x; i < 1024; i += blockDim.x)
        s_lut[i] = g_hilbert_lut.v[i];
    __syncthreads();
}

template <int BITS, typename U>
__device__ __forceinline__ U hilbert_key_lut(U x, U y,
                                             const uint16_t *s_lut) {
    constexpr int H = BITS / 2;
    uint32_t st = 0;
    U d = 0;
#pragma unroll
    for (int l = H - 4; l >= 0; l -= 4) {
        const uint32_t e = s_lut[st | ((uint32_t)(x >> l) & 15u) << 4 |
                                 ((uint32_t)(y >> l) & 15u)];
        d = (d << 8) | (U)(e & 255u);
        st = e & 0x300u;
    }
    return d;
}

// The key of one point (its coordinates already re-centred).
template <int BITS, bool HILBERT>
__device__ __forceinline__
    typename std::conditional<BITS == 32, uint32_t, uint64_t>::type
    point_key(double x, double y, double root0, double root1, double scale) {
    const double q0 = __dmul_rn(__dsub_rn(x, root0), scale);
    const double q1 = __dmul_rn(__dsub_rn(y, root1), scale);
    if constexpr (BITS == 32) {
        const uint32_t m0 = __double2uint_rz(q0), m1 = __double2uint_rz(q1);
        return HILBERT ? hilbert_key<32>(m0, m1)
                       : spread16(m0) | (spread16(m1) << 1);
    } else {
        const uint64_t m0 = __double2ull_rz(q0), m1 = __double2ull_rz(q1);
        return HILBERT ? hilbert_key<64>(m0, m1)
                       : spread32(m0) | (spread32(m1) << 1);
    }
}

// The same key with the Hilbert walk read from the staged table.
template <int BITS>
__device__ __forceinline__
    typename std::conditional<BITS == 32, uint32_t, uint64_t>::type
    point_key_hilbert_lut(double x, double y, double root0, double root1,
                          double scale, const uint16_t *s_lut) {
    const double q0 = __dmul_rn(__dsub_rn(x, root0), scale);
    const double q1 = __dmul_rn(__dsub_rn(y, root1), scale);
    if constexpr (BITS == 32) {
        const uint32_t m0 = __double2uint_rz(q0), m1 = __double2uint_rz(q1);
        return hilbert_key_lut<32>(m0, m1, s_lut);
    } else {
        const uint64_t m0 = __double2ull_rz(q0), m1 = __double2ull_rz(q1);
        return hilbert_key_lut<64>(m0, m1, s_lut);
    }
}

}  // namespace bh
