// launch_probe.cu — host cost of a kernel launch on this box (B200): empty
// kernel, an n = 150,000 axpy, and launch + spin-wait on a mapped host flag
// (what a harness dot's result wait looks like). Diagnostic only.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/launch_probe tools/cuda/launch_probe.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty() {}
__global__ void k_axpy(int n, double* y, double a, const double* x) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] += a * x[i];
}
__global__ void k_flag(volatile unsigned* f, unsigned v) {
    if (threadIdx.x == 0) *f = v;
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int n = 150000;
    double *x, *y;
    cudaMalloc(&x, n * 8);
    cudaMalloc(&y, n * 8);
    unsigned* hf;
    cudaHostAlloc(&hf, 64, cudaHostAllocMapped);
    unsigned* df;
    cudaHostGetDevicePointer(&df, hf, 0);
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    for (int w = 0; w < 100; ++w) k_empty<<<1, 32, 0, s>>>();
    cudaStreamSynchronize(s);
    const int R = 2000;
    auto t0 = now();
    for (int i = 0; i < R; ++i) k_empty<<<1, 32, 0, s>>>();
    auto t1 = now();
    cudaStreamSynchronize(s);
    std::printf("empty launch, host us/launch: %.2f\n", us(t0, t1) / R);
    t0 = now();
    for (int i = 0; i < R; ++i) k_axpy<<<(n + 255) / 256, 256, 0, s>>>(n, y, 0.5, x);
    t1 = now();
    cudaStreamSynchronize(s);
    auto t2 = now();
    std::printf("axpy launch, host us/launch: %.2f (incl. drain %.2f us/launch)\n", us(t0, t1) / R, us(t0, t2) / R);
    t0 = now();
    for (int i = 0; i < R; ++i) {
        k_axpy<<<(n + 255) / 256, 256, 0, s>>>(n, y, 0.5, x);
        cudaStreamSynchronize(s);
    }
    t1 = now();
    std::printf("axpy launch + stream sync: %.2f us\n", us(t0, t1) / R);
    t0 = now();
    for (int i = 1; i <= R; ++i) {
        k_flag<<<1, 32, 0, s>>>(df, static_cast<unsigned>(i));
        while (*reinterpret_cast<volatile unsigned*>(hf) != static_cast<unsigned>(i)) {
        }
    }
    t1 = now();
    std::printf("flag launch + host spin: %.2f us\n", us(t0, t1) / R);
    t0 = now();
    for (int i = 1; i <= R; ++i) {
        k_axpy<<<(n + 255) / 256, 256, 0, s>>>(n, y, 0.5, x);
        k_flag<<<1, 32, 0, s>>>(df, static_cast<unsigned>(i + R));
        while (*reinterpret_cast<volatile unsigned*>(hf) != static_cast<unsigned>(i + R)) {
        }
    }
    t1 = now();
    std::printf("axpy + flag launch + host spin: %.2f us\n", us(t0, t1) / R);
    return 0;
}
