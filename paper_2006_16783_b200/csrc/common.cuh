// Shared device/host helpers of the B200 siting engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace txs {

// ---- splitmix64 (stream semantics of proj/include/txsite/rng.hpp:9-36) -------
// The reference generator's state is a counter (state += gamma per draw,
// rng.hpp:14), so draw k of a stream is a pure function of (seed, k): lanes of
// a warp evaluate consecutive draws of one stream in parallel.
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t sm_finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// k-th (0-based) next() of SplitMix64(seed)
__host__ __device__ __forceinline__ uint64_t sm_draw(uint64_t seed, uint64_t k) {
    return sm_finalize(seed + (k + 1) * kGamma);
}
// mix_seed(a,b,c), rng.hpp:31-36
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t h = sm_draw(a, 0) ^ (b * 0xFF51AFD7ED558CCDull);
    return sm_draw(h, 0) ^ (c * 0xC4CEB9FE1A85EC53ull);
}

// ---- exact x % d for a runtime-invariant d (next_below, rng.hpp:21) ----------
// Round-up multiply-shift division (Granlund-Montgomery, "add" variant), exact
// for every 64-bit x and every d >= 2 that is not a power of two; the
// 64-bit '%' the reference uses compiles to a ~100-instruction software
// routine on the GPU.  Verified exhaustively-by-sampling in txs_selftest().
struct FastMod64 {
    uint64_t d;
    uint64_t magic;
    uint32_t shift;
    uint32_t pow2;   // d is a power of two: use the mask
};

__host__ __device__ __forceinline__ uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ uint64_t fm_div(const FastMod64& f, uint64_t x) {
    if (f.pow2) return x >> f.shift;
    const uint64_t q = umulhi64(f.magic, x);
    return (((x - q) >> 1) + q) >> f.shift;
}
__host__ __device__ __forceinline__ uint64_t fm_mod(const FastMod64& f, uint64_t x) {
    return x - fm_div(f, x) * f.d;
}

inline FastMod64 make_fastmod(uint64_t d) {
    FastMod64 f{d, 0, 0, 0};
    uint32_t l = 63 - (uint32_t)__builtin_clzll(d);
    if ((d & (d - 1)) == 0) { f.pow2 = 1; f.shift = l; return f; }
    const unsigned __int128 num = (unsigned __int128)1 << (64 + l);
    uint64_t pm = (uint64_t)(num / d);
    const uint64_t rem = (uint64_t)(num % d);
    pm += pm;
    const uint64_t twice = rem + rem;
    if (twice >= d || twice < rem) pm += 1;
    f.magic = pm + 1;
    f.shift = l;
    return f;
}

__host__ __device__ __forceinline__ int64_t floordiv64(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

// ---- bounds-checked build (make checked -> libtxsite_b200_checked.so) ---------
// Every global terrain load goes through zld(); with TXS_BOUNDS_CHECK it traps
// on an address outside the held terrain rows (compute-sanitizer is not
// available on the B200 pool, so the tests run edge-heavy workloads on this
// build instead).  Release builds compile zld() to a plain __ldg.
// Two ranges: the held terrain rows and (VIX global path) their column-major copy.
struct ZBounds { const int16_t* lo; const int16_t* hi; const int16_t* lo2; const int16_t* hi2; };
#ifdef TXS_BOUNDS_CHECK
static __device__ ZBounds g_zb;
__device__ __forceinline__ int zld(const int16_t* p) {
    if ((p < g_zb.lo || p >= g_zb.hi) && (p < g_zb.lo2 || p >= g_zb.hi2)) __trap();
    return __ldg(p);
}
inline void set_zbounds(const int16_t* lo, const int16_t* hi, cudaStream_t s, const int16_t* lo2 = nullptr,
                        const int16_t* hi2 = nullptr) {
    const ZBounds b{lo, hi, lo2, hi2};
    cudaMemcpyToSymbolAsync(g_zb, &b, sizeof(b), 0, cudaMemcpyHostToDevice, s);
}
#else
__device__ __forceinline__ int zld(const int16_t* p) { return __ldg(p); }
inline void set_zbounds(const int16_t*, const int16_t*, cudaStream_t, const int16_t* = nullptr,
                        const int16_t* = nullptr) {}
#endif

}  // namespace txs
