#pragma once
// ldst.cuh — L2 cache-policy loads for the SpMV kernels.
//
// The matrix is streamed once per SpMV (evict_first: do not let it push x out
// of L2); x is gathered at random (evict_last: keep it resident across the
// whole launch — Kronecker scale 22's x is 33.5 MB of the 126 MB L2).

#include <cstdint>

namespace b200 {

__device__ __forceinline__ std::uint64_t policy_evict_first() {
    std::uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ std::uint64_t policy_evict_last() {
    std::uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// streamed, read-once: no L1 allocation, L2 evict-first
__device__ __forceinline__ double ld_stream_f64(const double* a, std::uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}

__device__ __forceinline__ std::int32_t ld_stream_s32(const std::int32_t* a, std::uint64_t pol) {
    std::int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}

__device__ __forceinline__ std::int64_t ld_stream_s64(const std::int64_t* a, std::uint64_t pol) {
    long long v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
    return v;
}

__device__ __forceinline__ std::int64_t ld_stream_idx(const std::int32_t* a, std::uint64_t pol) {
    return ld_stream_s32(a, pol);
}
__device__ __forceinline__ std::int64_t ld_stream_idx(const std::int64_t* a, std::uint64_t pol) {
    return ld_stream_s64(a, pol);
}

// gathered, reused: read-only path, L2 evict-last
__device__ __forceinline__ double ld_gather_f64(const double* a, std::uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}

}  // namespace b200
