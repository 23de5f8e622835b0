// generate_fractal on the device — decision D10.
//
// Integer diamond-square on a (2^k+1)^2 int32 canvas in HBM (config 4: 65537^2
// = 17.2 GB, freed afterwards), one diamond and one square kernel per level.
// Every value is an integer function of (seed, y, x, level), so the result is
// bit-identical to the CPU restatement in oracle/oracle.cpp.
#include <cmath>
#include <vector>

#include "ctx.hpp"

namespace txs {
namespace {

constexpr int64_t kA0 = (int64_t)1 << 20;

__device__ __forceinline__ int32_t disp(uint64_t seed, int64_t y, int64_t x, int64_t A, const FastMod64& m) {
    if (A <= 0) return 0;
    const uint64_t h = sm_draw(mix_seed(seed, (uint64_t)y, (uint64_t)x), 0);
    return (int32_t)((int64_t)fm_mod(m, h) - A);
}

__global__ void k_corners(int32_t* cv, int64_t N, uint64_t seed, int64_t A, FastMod64 m) {
    const int i = threadIdx.x;
    if (i >= 4) return;
    const int64_t y = (i & 2) ? N - 1 : 0, x = (i & 1) ? N - 1 : 0;
    cv[y * N + x] = disp(seed, y, x, A, m);
}

__global__ void k_diamond(int32_t* __restrict__ cv, int64_t N, int64_t s, int64_t nsq, uint64_t seed,
                          int64_t A, FastMod64 m) {
    const int64_t h = s >> 1, total = nsq * nsq;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / nsq, j = t - i * nsq;
        const int64_t y = h + i * s, x = h + j * s;
        const int64_t sum = (int64_t)cv[(y - h) * N + x - h] + cv[(y - h) * N + x + h] +
                            cv[(y + h) * N + x - h] + cv[(y + h) * N + x + h];
        cv[y * N + x] = (int32_t)(floordiv64(sum, 4) + disp(seed, y, x, A, m));
    }
}

// square step: rows iy = 0..(N-1)/h; odd rows start at x = 0, even at x = h; step s
__global__ void k_square(int32_t* __restrict__ cv, int64_t N, int64_t s, uint64_t seed, int64_t A, FastMod64 m) {
    const int64_t h = s >> 1, nrow = (N - 1) / h + 1, per = (N - 1) / s + 1, total = nrow * per;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t iy = t / per, jx = t - iy * per;
        const int64_t y = iy * h, x = ((iy & 1) ? 0 : h) + jx * s;
        if (x >= N) continue;
        int64_t sum = 0, cnt = 0;
        if (y - h >= 0) { sum += cv[(y - h) * N + x]; ++cnt; }
        if (y + h < N) { sum += cv[(y + h) * N + x]; ++cnt; }
        if (x - h >= 0) { sum += cv[y * N + x - h]; ++cnt; }
        if (x + h < N) { sum += cv[y * N + x + h]; ++cnt; }
        cv[y * N + x] = (int32_t)(floordiv64(sum, cnt) + disp(seed, y, x, A, m));
    }
}

// crop held rows [row0, row0 + rows) of the canvas into z (rows x ncols)
__global__ void k_crop(const int32_t* __restrict__ cv, int64_t N, int16_t* __restrict__ z, int64_t row0, int64_t rows,
                       int64_t ncols, int64_t zmin, int64_t zmax) {
    const int64_t range = zmax - zmin, mid = zmin + range / 2, total = rows * ncols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = row0 + t / ncols, x = t % ncols;
        int64_t v = mid + floordiv64((int64_t)cv[y * N + x] * range, (int64_t)1 << 21);
        v = v < zmin ? zmin : (v > zmax ? zmax : v);
        z[t] = (int16_t)v;
    }
}

__global__ void k_fill_rows(int16_t* z, int64_t begin, int64_t end, int16_t v) {
    for (int64_t t = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < end; t += (int64_t)gridDim.x * blockDim.x)
        z[t] = v;
}

int grid_for(int64_t work, int sms) {
    const int64_t b = (work + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sms * 32));
}

}  // namespace

txs_status launch_generate(txs_ctx* c, int64_t nrows, int64_t ncols, double roughness, uint64_t seed,
                           int32_t zmin, int32_t zmax) {
    int k = 1;
    while (((int64_t)1 << k) + 1 < std::max(nrows, ncols)) ++k;
    const int64_t N = ((int64_t)1 << k) + 1;
    std::vector<int64_t> amp(k + 1);
    double a = (double)kA0;
    for (int i = 0; i <= k; ++i) { a *= roughness; amp[i] = (int64_t)std::floor(a); }
    int32_t* cv = nullptr;
    TXS_CUDA(c, "read", cudaMallocAsync((void**)&cv, sizeof(int32_t) * N * N, c->stream));
    auto mod_for = [](int64_t A) { return make_fastmod((uint64_t)(2 * std::max<int64_t>(A, 1) + 1)); };
    k_corners<<<1, 32, 0, c->stream>>>(cv, N, seed, amp[0], mod_for(amp[0]));
    TXS_LAUNCHED(c, "read");
    for (int L = 0; L < k; ++L) {
        const int64_t s = (int64_t)1 << (k - L), nsq = (N - 1) / s, A = amp[L + 1];
        k_diamond<<<grid_for(nsq * nsq, c->num_sms), 256, 0, c->stream>>>(cv, N, s, nsq, seed, A, mod_for(A));
        TXS_LAUNCHED(c, "read");
        const int64_t h = s / 2, work = ((N - 1) / h + 1) * ((N - 1) / s + 1);
        k_square<<<grid_for(work, c->num_sms), 256, 0, c->stream>>>(cv, N, s, seed, A, mod_for(A));
        TXS_LAUNCHED(c, "read");
    }
    k_crop<<<grid_for(c->z_rows * ncols, c->num_sms), 256, 0, c->stream>>>(cv, N, c->d_z, c->z_off, c->z_rows, ncols, zmin, zmax);
    TXS_LAUNCHED(c, "read");
    TXS_CUDA(c, "read", cudaFreeAsync(cv, c->stream));
    return TXS_OK;
}

txs_status launch_fill_rows(txs_ctx* c, int64_t rb, int64_t re, int16_t v) {
    if (re <= rb) return TXS_OK;
    k_fill_rows<<<grid_for((re - rb) * c->ncols, c->num_sms), 256, 0, c->stream>>>(c->d_z, rb * c->ncols, re * c->ncols, v);
    TXS_LAUNCHED(c, "read");
    TXS_CUDA(c, "read", cudaStreamSynchronize(c->stream));
    return TXS_OK;
}

}  // namespace txs
