// Microbenchmark: does cp.async.bulk.prefetch.L2 of a buffer make a following read kernel hit in L2?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void prefetch_kernel(const uint8_t* p, size_t bytes, uint32_t chunk) {
  size_t n = bytes / chunk;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + i * chunk), "r"(chunk) : "memory");
}
__global__ void read_kernel(const uint4* p, size_t n, uint4* out) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t st = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * st) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i + u * st < n ? __ldcg(p + i + u * st) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  if (acc.x == 0x12345678) out[0] = acc;
}
__global__ void spin_kernel(long long cyc) {
  long long t0 = clock64();
  while (clock64() - t0 < cyc) {}
}
__global__ void flush_kernel(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = make_uint4(i, 0, 0, 0);
}

int main() {
  const size_t fl = 512ull << 20;
  uint8_t* buf; uint4* fbuf; uint4* out;
  cudaMalloc(&buf, 64ull << 20); cudaMalloc(&fbuf, fl); cudaMalloc(&out, 64);
  cudaMemset(buf, 1, 64ull << 20);
  cudaEvent_t e1, e2; cudaEventCreate(&e1); cudaEventCreate(&e2);
  auto timed_read = [&](size_t bytes) {
    cudaEventRecord(e1);
    read_kernel<<<148 * 4, 512>>>((const uint4*)buf, bytes / 16, out);
    cudaEventRecord(e2);
    cudaEventSynchronize(e2);
    float ms; cudaEventElapsedTime(&ms, e1, e2);
    return ms * 1e3f;
  };
  for (size_t mb : {4, 8, 16, 32, 48, 64}) {
    const size_t bytes = mb << 20;
    for (int rep = 0; rep < 2; ++rep) {
      flush_kernel<<<592, 512>>>(fbuf, fl / 16); cudaDeviceSynchronize();
      float cold = timed_read(bytes);
      float warm = timed_read(bytes);
      flush_kernel<<<592, 512>>>(fbuf, fl / 16); cudaDeviceSynchronize();
      prefetch_kernel<<<148, 32>>>(buf, bytes, 16384);
      spin_kernel<<<1, 32>>>(400000);
      float pf = timed_read(bytes);
      flush_kernel<<<592, 512>>>(fbuf, fl / 16); cudaDeviceSynchronize();
      prefetch_kernel<<<148, 32>>>(buf, bytes, 1024);
      spin_kernel<<<1, 32>>>(400000);
      float pf1 = timed_read(bytes);
      printf("%2zu MB: cold %.1f us (%.0f GB/s) warm %.1f us (%.0f GB/s) after prefetch 16K %.1f us, 1K %.1f us\n", mb, cold,
             bytes / (cold * 1e-6) / 1e9, warm, bytes / (warm * 1e-6) / 1e9, pf, pf1);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
