#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
struct Big { int v[100]; };
__global__ void k0(int* p) { if (p && threadIdx.x == 1234567) *p = 1; }
__global__ void k1(Big b, int* p) { if (p && threadIdx.x == 1234567) *p = b.v[3]; }
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* d; cudaMalloc(&d, 4);
  Big b{};
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 10000; ++i) k0<<<1, 32, 0, st>>>(d);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto t2 = std::chrono::steady_clock::now();
    for (int i = 0; i < 10000; ++i) k1<<<148, 256, 0, st>>>(b, d);
    auto t3 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto t4 = std::chrono::steady_clock::now();
    for (int i = 0; i < 1000; ++i) { k0<<<1, 32, 0, st>>>(d); cudaStreamSynchronize(st); }
    auto t5 = std::chrono::steady_clock::now();
    for (int i = 0; i < 1000; ++i) cudaMemsetAsync(d, 0, 4, st);
    auto t6 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    printf("launch small %.2f us, launch 400B param 148x256 %.2f us (gpu drain %.1f us per), launch+sync %.2f us, memset %.2f us\n",
           us(t0, t1) / 10000, us(t2, t3) / 10000, us(t2, t4) / 10000, us(t4, t5) / 1000, us(t5, t6) / 1000);
  }
  return 0;
}
