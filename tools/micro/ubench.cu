// Instruction-throughput microbenchmarks on sm_100a (development tool).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CHAINS>
__global__ void k_hmma(float* out, int iters, uint32_t s) {
  float d[CHAINS][4];
  for (int c = 0; c < CHAINS; ++c) for (int e = 0; e < 4; ++e) d[c][e] = 0.f;
  uint32_t a = s ^ threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) mma(d[c], a, a + 1, a + 2, a + 3, a + c, a);
  }
  float t = 0; for (int c = 0; c < CHAINS; ++c) t += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (t == 12345.f) out[0] = t;
}

template <int OP>
__global__ void k_alu(uint32_t* out, int iters, uint32_t s) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = s + threadIdx.x * 7 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) v[i] = v[i] >> (3 + i);                         // SHF
      if (OP == 1) { uint32_t d; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(v[i]), "r"(1u << (20 + i))); v[i] = d + 1; }      // IMAD.HI
      if (OP == 2) { uint32_t d; asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v[i]), "r"(0x0f0f0f0fu), "r"(v[(i+1)&7])); v[i] = d; }
      if (OP == 3) { __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&v[i]); __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162*>(&v[(i+3)&7]);
                     x = __hsub2(x, y); v[i] = *reinterpret_cast<uint32_t*>(&x); }
    }
  }
  uint32_t t = 0; for (int i = 0; i < 8; ++i) t ^= v[i];
  if (t == 0x12345678u) out[0] = t;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  float* of; uint32_t* ou; cudaMalloc(&of, 64); cudaMalloc(&ou, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    float ms1 = timeit([&] { k_hmma<1><<<sms, warps * 32>>>(of, iters, 1); });
    float ms4 = timeit([&] { k_hmma<4><<<sms, warps * 32>>>(of, iters, 1); });
    double n1 = (double)sms * warps * iters * 1, n4 = (double)sms * warps * iters * 4;
    printf("HMMA m16n8k16 bf16: warps/SM %2d  1 chain: %.2f ns/inst/SM (%.1f TFLOPS)   4 chains: %.2f ns/inst/SM (%.1f TFLOPS)\n",
           warps, ms1 * 1e6 / (n1 / sms), n1 * 4096 / ms1 / 1e9, ms4 * 1e6 / (n4 / sms), n4 * 4096 / ms4 / 1e9);
  }
  const char* names[4] = {"SHF", "IMAD.HI", "LOP3", "HADD2.BF16"};
  for (int op = 0; op < 4; ++op) {
    for (int warps : {8, 32}) {
      float ms;
      if (op == 0) ms = timeit([&] { k_alu<0><<<sms, warps * 32>>>(ou, iters, 1); });
      if (op == 1) ms = timeit([&] { k_alu<1><<<sms, warps * 32>>>(ou, iters, 1); });
      if (op == 2) ms = timeit([&] { k_alu<2><<<sms, warps * 32>>>(ou, iters, 1); });
      if (op == 3) ms = timeit([&] { k_alu<3><<<sms, warps * 32>>>(ou, iters, 1); });
      double n = (double)warps * iters * 8;   // warp-instructions per SM
      printf("%-10s warps/SM %2d: %.3f cycles-equiv ns per warp-inst per SM -> %.2f warp-inst/ns/SM\n", names[op], warps,
             ms * 1e6 / n, n / (ms * 1e6));
    }
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
