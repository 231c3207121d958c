// Throughput of the decode's integer instructions on one SM (B200): PRMT, LOP3,
// IMAD.HI, IMAD.SHL, and mixes -- warp-instructions per cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_alu tools/ubench_alu.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(unsigned* out, unsigned seed, int iters) {
  unsigned r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = seed * (threadIdx.x + i);
  const unsigned c1 = seed | 0x7604, c2 = seed ^ 0x44444444u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(c2), "r"(c1));
      if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(r[i]) : "r"(c2), "r"(c1));
      if (OP == 2) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(c1));
      if (OP == 3) asm volatile("shl.b32 %0, %0, 2;" : "+r"(r[i]));
      if (OP == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(c1));
      if (OP == 6) asm volatile("shr.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(c1 & 15));
      if (OP == 7) asm volatile("shf.r.wrap.b32 %0, %0, %1, 16;" : "+r"(r[i]) : "r"(c2));
      if (OP == 8) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(c1), "r"(c2));
      if (OP == 9) asm volatile("bfe.u32 %0, %0, 16, 16;" : "+r"(r[i]));
      if (OP == 10) { unsigned x = r[i]; asm volatile("" : "+r"(x)); r[i] = (x >> 16) + c2; }  // LEA.HI?
      if (OP == 11) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(c1));
      if (OP == 12) asm volatile("ld.shared.u32 %0, [%0];" : "+r"(r[i]));
      if (OP >= 20) {  // pairs: PRMT + X (X on the same pipe -> 2/cycle/SM, else up to 4)
        asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(c2), "r"(c1));
        if (OP == 20) asm volatile("shr.u32 %0, %0, %1;" : "+r"(r[(i + 4) & 7]) : "r"(c1 & 15));
        if (OP == 21) { unsigned x = r[(i + 4) & 7]; asm volatile("" : "+r"(x)); r[(i + 4) & 7] = (x >> 16) + c2; }
        if (OP == 22) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(r[(i + 4) & 7]) : "r"(c1));
        if (OP == 23) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[(i + 4) & 7]) : "r"(c1), "r"(c2));
        if (OP == 24) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[(i + 4) & 7]) : "r"(c1));
        if (OP == 25) asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(r[(i + 4) & 7]) : "r"(c2), "r"(c1));
        if (OP == 26) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r[(i + 4) & 7]) : "r"((threadIdx.x & 31) * 4));
      }
      if (OP == 5) {  // decode mix: PRMT PRMT LOP3 PRMT + mul.hi
        asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(c2), "r"(c1));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(r[i]) : "r"(c2), "r"(c1));
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(c1));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = unsigned(t1 - t0);
}
int main() {
  unsigned* d;
  cudaMalloc(&d, (1 << 22) * 4);
  const char* pn[] = {"prmt+shr", "prmt+lea.hi", "prmt+mul.hi", "prmt+mad.lo", "prmt+add", "prmt+lop3", "prmt+lds"};
  for (int op = 20; op < 27; ++op) {
    auto run = [&] {
      switch (op) {
        case 20: k<20><<<1, 512>>>(d, 3, 4096); break;
        case 21: k<21><<<1, 512>>>(d, 3, 4096); break;
        case 22: k<22><<<1, 512>>>(d, 3, 4096); break;
        case 23: k<23><<<1, 512>>>(d, 3, 4096); break;
        case 24: k<24><<<1, 512>>>(d, 3, 4096); break;
        case 25: k<25><<<1, 512>>>(d, 3, 4096); break;
        default: k<26><<<1, 512>>>(d, 3, 4096); break;
      }
    };
    run(); run();
    cudaError_t e = cudaDeviceSynchronize();
    unsigned cyc;
    cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
    printf("%-14s %.3f warp-inst/cycle/SM %s\n", pn[op - 20], 16.0 * 4096 * 16 / cyc, cudaGetErrorString(e));
  }
  const char* names[] = {"prmt", "lop3", "mul.hi", "shl", "add", "mix(prmt,lop3,mulhi)", "shr", "shf.r", "mad.lo", "bfe", "x>>16+y", "mul.lo", "lds"};
  const int insts[] = {1, 1, 1, 1, 1, 3, 1, 1, 1, 1, 1, 1, 1};
  for (int warps = 16; warps <= 16; warps *= 2) {
    for (int op = 0; op < 13; ++op) {
      if (op == 3) continue;
      const int iters = 4096;
      auto run = [&] {
        switch (op) {
          case 0: k<0><<<1, warps * 32>>>(d, 3, iters); break;
          case 1: k<1><<<1, warps * 32>>>(d, 3, iters); break;
          case 2: k<2><<<1, warps * 32>>>(d, 3, iters); break;
          case 3: k<3><<<1, warps * 32>>>(d, 3, iters); break;
          case 4: k<4><<<1, warps * 32>>>(d, 3, iters); break;
          case 5: k<5><<<1, warps * 32>>>(d, 3, iters); break;
          case 6: k<6><<<1, warps * 32>>>(d, 3, iters); break;
          case 7: k<7><<<1, warps * 32>>>(d, 3, iters); break;
          case 8: k<8><<<1, warps * 32>>>(d, 3, iters); break;
          case 9: k<9><<<1, warps * 32>>>(d, 3, iters); break;
          case 10: k<10><<<1, warps * 32>>>(d, 3, iters); break;
          case 11: k<11><<<1, warps * 32>>>(d, 3, iters); break;
          default: k<12><<<1, warps * 32>>>(d, 3, iters); break;
        }
      };
      run();
      run();
      cudaDeviceSynchronize();
      unsigned cyc;
      cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
      const double winst = double(warps) * iters * 8 * insts[op];
      printf("warps %2d %-22s %.3f warp-inst/cycle/SM\n", warps, names[op], winst / cyc);
    }
  }
  return 0;
}
