// host_calls.cu — per-call host cost of the C-ABI harness entry points against
// the raw CUDA API floor (one B200). Build + run:
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/host_calls.cu \
//        -Lpaper_2001_07938_b200 -llilac_b200 -Xlinker -rpath,$PWD/paper_2001_07938_b200 -o /tmp/host_calls
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "lilac_b200.h"

using Clock = std::chrono::steady_clock;

__global__ void k_empty() {}

template <typename F>
double per_call_us(int n, F&& f) {
    for (int i = 0; i < 10; ++i) f();
    cudaDeviceSynchronize();
    auto t0 = Clock::now();
    for (int i = 0; i < n; ++i) f();
    const double us = std::chrono::duration<double, std::micro>(Clock::now() - t0).count() / n;
    cudaDeviceSynchronize();
    return us;
}

static double* page_aligned(std::size_t n) {
    void* p = mmap(nullptr, (n * 8 + 4095) / 4096 * 4096, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    return static_cast<double*>(p);
}

int main(int argc, char** argv) {
    const std::int64_t n = argc > 1 ? std::atoll(argv[1]) : 150000;
    b200_init(0);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double *d1, *d2, *hp;
    cudaMalloc(&d1, n * 8);
    cudaMalloc(&d2, n * 8);
    cudaMallocHost(&hp, 64);
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    std::printf("raw: launch empty kernel      %.2f us\n", per_call_us(2000, [&] { k_empty<<<1, 32, 0, s>>>(); }));
    std::printf("raw: memcpyAsync D2D %lld B   %.2f us\n", (long long)(n * 8),
                per_call_us(2000, [&] { cudaMemcpyAsync(d1, d2, n * 8, cudaMemcpyDeviceToDevice, s); }));
    std::printf("raw: eventRecord              %.2f us\n", per_call_us(2000, [&] { cudaEventRecord(ev, s); }));
    std::printf("raw: memsetAsync 64 B         %.2f us\n", per_call_us(2000, [&] { cudaMemsetAsync(d1, 0, 64, s); }));
    std::printf("raw: empty kernel + sync      %.2f us\n", per_call_us(2000, [&] {
                    k_empty<<<1, 32, 0, s>>>();
                    cudaStreamSynchronize(s);
                }));
    std::printf("raw: D2H 8 B (pinned) + sync  %.2f us\n", per_call_us(2000, [&] {
                    cudaMemcpyAsync(hp, d1, 8, cudaMemcpyDeviceToHost, s);
                    cudaStreamSynchronize(s);
                }));
    double res = 0;
    std::printf("raw: D2H 8 B (pageable)+sync  %.2f us\n", per_call_us(2000, [&] {
                    cudaMemcpyAsync(&res, d1, 8, cudaMemcpyDeviceToHost, s);
                    cudaStreamSynchronize(s);
                }));

    double *x = page_aligned(n), *y = page_aligned(n), *z = page_aligned(n);
    for (std::int64_t i = 0; i < n; ++i) x[i] = 1.0 + i % 7, y[i] = 0.5, z[i] = 0.0;
    for (const char* mode : {"eager", "lazy"}) {
        b200_set_writeback(mode);
        std::printf("[%s] b200_axpy n=%lld          %.2f us\n", mode, (long long)n,
                    per_call_us(2000, [&] { b200_axpy(n, z, 0.5, x); }));
        std::printf("[%s] b200_xpay                 %.2f us\n", mode,
                    per_call_us(2000, [&] { b200_xpay(n, y, 0.5, z); }));
        std::printf("[%s] b200_dot                  %.2f us\n", mode,
                    per_call_us(2000, [&] { b200_dot(&res, n, x, z); }));
        std::printf("[%s] axpy+dot (CG pair)        %.2f us\n", mode, per_call_us(1000, [&] {
                        b200_axpy(n, z, 0.5, x);
                        b200_dot(&res, n, z, z);
                    }));
        b200_host_sync(nullptr, 0);
    }
    // a banded SpMV (7 nonzeros per row)
    std::vector<std::int64_t> rp(n + 1), ci;
    std::vector<double> val;
    for (std::int64_t i = 0; i < n; ++i) {
        rp[i] = static_cast<std::int64_t>(ci.size());
        for (std::int64_t k = -3; k <= 3; ++k)
            if (i + k >= 0 && i + k < n) ci.push_back(i + k), val.push_back(1.0 / (1 + (k < 0 ? -k : k)));
    }
    rp[n] = static_cast<std::int64_t>(ci.size());
    for (const char* mode : {"eager", "lazy"}) {
        b200_set_writeback(mode);
        std::printf("[%s] b200_spmv_csr (7/row)     %.2f us\n", mode, per_call_us(2000, [&] {
                        b200_spmv_csr(n, z, rp.data(), val.data(), x, ci.data());
                    }));
        b200_host_sync(nullptr, 0);
    }
    b200_shutdown();
    return 0;
}
