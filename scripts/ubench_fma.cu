// Experiments only: issue cost of the FP32 instruction forms the rollout uses, on this
// B200 (scalar FFMA with 3 registers / an immediate / a constant-bank operand, FMUL,
// FADD, packed FFMA2 / FMUL2 / FADD2).  Every thread runs 8 independent chains of one
// form; the result is warp instructions per cycle per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench_fma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float c_k[4];

template <int OP>
__global__ void __launch_bounds__(256) bench(float* out, int iters, float a, float b) {
  float x[8], y[8];
  float2 u[8], v[8];
  uint32_t w[8], h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = a + i * threadIdx.x;
    y[i] = b - i;
    u[i] = make_float2(x[i], y[i]);
    v[i] = make_float2(y[i], x[i]);
    w[i] = threadIdx.x * 7919u + i;
    h[i] = w[i] ^ 0x9E3779B9u;
  }
  const float2 kk = make_float2(a * 0.5f, b * 0.25f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) x[i] = fmaf(x[i], y[i], x[(i + 1) & 7]);            // FFMA, 3 registers
        if (OP == 1) x[i] = fmaf(x[i], 1.0001f, y[i]);                   // FFMA, immediate
        if (OP == 2) x[i] = fmaf(x[i], c_k[0], y[i]);                    // FFMA, constant bank
        if (OP == 3) x[i] = x[i] * y[i];                                 // FMUL, 2 registers
        if (OP == 4) x[i] = x[i] + y[i];                                 // FADD, 2 registers
        if (OP == 5) u[i] = __ffma2_rn(u[i], v[i], u[(i + 1) & 7]);      // FFMA2, 3 pairs
        if (OP == 6) u[i] = __fmul2_rn(u[i], v[i]);                      // FMUL2
        if (OP == 7) u[i] = __fadd2_rn(u[i], v[i]);                      // FADD2
        if (OP == 8) u[i] = __ffma2_rn(u[i], kk, v[i]);                  // FFMA2, loop-invariant pair
        if (OP == 9) x[i] = fmaf(x[i], y[i], 0.5f);                      // FFMA, imm addend
        if (OP == 10) {                                                   // IMAD.WIDE (Philox round product)
          const uint64_t pr = (uint64_t)w[i] * 0xD2511F53u;
          w[i] = (uint32_t)(pr >> 32) ^ h[i];
          h[i] = (uint32_t)pr;
        }
        if (OP == 11) w[i] = w[i] ^ h[i] ^ 0x9E3779B9u;                  // LOP3
        if (OP == 12) x[i] = __sinf(x[i]);                               // MUFU.SIN (+ FMUL.RZ)
        if (OP == 13) u[i] = __ffma2_rn(u[i], v[i], make_float2(0.5f, 0.5f));  // FFMA2, imm addend
        if (OP == 15) {                                                   // Philox round, hi via mul.hi, lo via mul.lo
          uint32_t h0, l0, h1, l1;
          asm("mul.hi.u32 %0, %1, 0xD2511F53;" : "=r"(h0) : "r"(w[i]));
          asm("mul.lo.u32 %0, %1, 0xD2511F53;" : "=r"(l0) : "r"(w[i]));
          asm("mul.hi.u32 %0, %1, 0xCD9E8D57;" : "=r"(h1) : "r"(h[i]));
          asm("mul.lo.u32 %0, %1, 0xCD9E8D57;" : "=r"(l1) : "r"(h[i]));
          w[i] = h1 ^ l0 ^ 0x12345u;
          h[i] = h0 ^ l1 ^ 0x6789u;
        }
        if (OP == 14) {                                                   // Philox round: 2 x IMAD.WIDE + 2 x LOP3
          const uint64_t p0 = (uint64_t)w[i] * 0xD2511F53u, p1 = (uint64_t)h[i] * 0xCD9E8D57u;
          w[i] = (uint32_t)(p1 >> 32) ^ (uint32_t)p0 ^ 0x12345u;
          h[i] = (uint32_t)(p0 >> 32) ^ (uint32_t)p1 ^ 0x6789u;
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + u[i].x + u[i].y + (float)(w[i] ^ h[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, float* d, int sms, int blocks_per_sm, int threads) {
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bench<OP><<<sms * blocks_per_sm, threads>>>(d, 10, 1.f, 2.f);
  cudaEventRecord(e0);
  bench<OP><<<sms * blocks_per_sm, threads>>>(d, iters, 1.f, 2.f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int mhz;
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
  const double warp_inst = (double)sms * blocks_per_sm * (threads / 32) * iters * 64.0;
  const double cycles = ms * 1e-3 * 1965e6;  // at clocks.max.sm
  printf("%-28s warps/SMSP %2d: %.3f warp-inst/cycle/SMSP (%.3f ms)\n", name, blocks_per_sm * threads / 128,
         warp_inst / (sms * 4.0) / cycles, ms);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float h[4] = {1.0001f, 0.f, 0.f, 0.f};
  cudaMemcpyToSymbol(c_k, h, sizeof h);
  float* d;
  cudaMalloc(&d, sms * 8 * 256 * sizeof(float));
  for (int bps : {4}) {
    run<0>("FFMA r,r,r", d, sms, bps, 256);
    run<1>("FFMA r,imm,r", d, sms, bps, 256);
    run<2>("FFMA r,c[],r", d, sms, bps, 256);
    run<9>("FFMA r,r,imm", d, sms, bps, 256);
    run<3>("FMUL r,r", d, sms, bps, 256);
    run<4>("FADD r,r", d, sms, bps, 256);
    run<5>("FFMA2 rr,rr,rr", d, sms, bps, 256);
    run<8>("FFMA2 rr,kk(inv),rr", d, sms, bps, 256);
    run<6>("FMUL2 rr,rr", d, sms, bps, 256);
    run<7>("FADD2 rr,rr", d, sms, bps, 256);
    run<13>("FFMA2 rr,rr,imm", d, sms, bps, 256);
    run<10>("IMAD.WIDE + LOP3", d, sms, bps, 256);
    run<14>("Philox round (4 instr)", d, sms, bps, 256);
    run<15>("Philox round hi/lo split", d, sms, bps, 256);
    run<12>("__sinf", d, sms, bps, 256);
  }
  return 0;
}
