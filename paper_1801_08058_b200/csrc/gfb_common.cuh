// Shared device helpers for the gfb200 kernels (sm_100a).
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

#include "gfb200.h"

// Loops over digits / program words: kept rolled in the generic kernels,
// unrolled (and folded) when the structure is a compile-time constant.
#ifdef __CUDACC_RTC__
#define GFB_LOOP _Pragma("unroll")
#else
#define GFB_LOOP _Pragma("unroll 1")
#endif

namespace gfb {

constexpr uint64_t kOffsetMask = (uint64_t(1) << 56) - 1;

// Resolve a GFB_REF through the executable's device pointer table.
template <typename T>
__device__ __forceinline__ T* resolve(const void* const* tab, uint64_t ref) {
    return reinterpret_cast<T*>(static_cast<char*>(const_cast<void*>(tab[ref >> 56])) + (ref & kOffsetMask));
}

// idx / d for idx < 2^31: (idx * mul) >> 32 >> sh, mul == 0 meaning d == 1
// (Granlund-Montgomery with a 31-bit dividend; see compiler.magic_u31).
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t mul, uint32_t sh) {
    return mul ? (__umulhi(n, mul) >> sh) : n;
}

__device__ __forceinline__ uint32_t digit_coord(const gfb_digit& d, uint32_t o, uint32_t r) {
    uint32_t n = d.src ? r : o;
    uint32_t q = fast_div(n, (uint32_t)d.div_mul, d.div_sh);
    if (d.mod) q -= fast_div(q, (uint32_t)d.mod_mul, d.mod_sh) * d.mod;
    return q;
}

__device__ __forceinline__ uint32_t leaf_offset(const gfb_leaf& L, uint32_t o, uint32_t r) {
    uint32_t off = 0;
    const int n = L.ndig;
    GFB_LOOP
    for (int i = 0; i < n; ++i) off += digit_coord(L.dig[i], o, r) * (uint32_t)L.dig[i].stride;
    return off;
}

}  // namespace gfb
