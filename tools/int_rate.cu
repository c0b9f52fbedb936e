// int_rate.cu -- INT32-pipe issue-rate microbenchmark for the hull DP's roofline (SURVEY 8(d):
// "Microbenchmark the sm_100 INT32 rate ... do not assume"; VERDICT r1 "Measure the ALU roofline").
//
// Each thread runs 8 independent dependency chains of one instruction class for ITER iterations;
// every block records clock64() and %globaltimer around its loop, which gives the SM clock
// under load; ops per SM-clock = thread-ops / (event time x that clock x SMs).
// The SASS each variant compiles to is checked with cuobjdump (tools/int_rate_sass.txt).
//
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/int_rate tools/int_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define ITER 65536
#define CH 8

enum Op { IADD3, LOP3, IMAD, ISETP_SEL, IMADWIDE, MIX_ALU_FMA, LDS32, SHFL, VIMNMX };
static const char* NAMES[] = {"IADD3 (2x add.s32)", "LOP3 (lop3.b32)", "IMAD (mad.lo.s32)",
                              "ISETP+SEL (setp+selp)", "IMAD.WIDE+IADD3 pair",
                              "IADD3+IMAD 1:1 mix", "LDS.32 (ld.shared.b32)",
                              "SHFL.IDX (shfl.sync)", "VIMNMX3 (2x min.s32)"};

template <int OP>
__global__ void __launch_bounds__(256) bench(int* out, long long* cyc, int seed) {
  __shared__ int sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 256) sm[i] = (i * 7 + seed) & 1023;
  __syncthreads();
  int r[CH];
  long long w[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    r[c] = threadIdx.x * 13 + c + seed;
    w[c] = r[c];
  }
  // per-thread (non-uniform) operands: uniform ones would cost a UR -> R move per use
  const int a = (seed | 1) + (int)(threadIdx.x & 2), b = seed * 3 + 5 + (int)(threadIdx.x & 4);
  int bc[CH], bm[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    bc[c] = b + c * (int)(threadIdx.x | 1);
    bm[c] = b - c * (int)(threadIdx.x | 1);
  }
  __syncthreads();
  long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == IADD3)   // two PTX adds of distinct registers: one 3-input IADD3
        asm volatile("add.s32 %0, %0, %1; add.s32 %0, %0, %2;" : "+r"(r[c]) : "r"(a), "r"(bc[c]));
      if (OP == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[c]) : "r"(a), "r"(bc[c]));
      if (OP == IMAD) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
      if (OP == ISETP_SEL)
        asm volatile("{.reg .pred p; setp.lt.s32 p, %0, %1; selp.s32 %0, %2, %0, p;}"
                     : "+r"(r[c]) : "r"(a), "r"(b));
      if (OP == IMADWIDE)
        asm volatile("{.reg .b64 t; .reg .b32 lo, hi; mul.wide.s32 t, %0, %1; mov.b64 {lo, hi}, t;"
                     " add.s32 %0, lo, hi;}" : "+r"(r[c]) : "r"(bc[c]));
      if (OP == MIX_ALU_FMA) {
        asm volatile("add.s32 %0, %0, %1;" : "+r"(r[c]) : "r"(a));
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
      }
      if (OP == LDS32) {
        const unsigned addr = (unsigned)__cvta_generic_to_shared(sm) + ((r[c] & 1023) << 2);
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(r[c]) : "r"(addr));
      }
      if (OP == SHFL) asm volatile("shfl.sync.idx.b32 %0, %0, %1, 31, -1;" : "+r"(r[c]) : "r"(a & 31));
      if (OP == VIMNMX)   // two PTX mins: one 3-input VIMNMX3
        asm volatile("min.s32 %0, %0, %1; min.s32 %0, %0, %2;" : "+r"(r[c]) : "r"(bc[c]), "r"(bm[c]));
    }
  }
  const long long t1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += r[c] + (int)w[c];
  out[blockIdx.x * 256 + threadIdx.x] = s;
  if (threadIdx.x == 0) {
    cyc[2 * blockIdx.x] = t1 - t0;
    cyc[2 * blockIdx.x + 1] = g1 - g0;   // ns: clock64 ticks / ns = the SM clock in GHz
  }
}

template <int OP>
static double run(int sms, int bps, int* out, long long* cyc, long long* hcyc, float* ms,
                  double* ghz) {
  const int nb = sms * bps;
  bench<OP><<<nb, 256>>>(out, cyc, 1);   // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<nb, 256>>>(out, cyc, 3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaMemcpy(hcyc, cyc, 2 * nb * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0, ns = 0;
  for (int i = 0; i < nb; ++i) {
    mean += (double)hcyc[2 * i];
    ns += (double)hcyc[2 * i + 1];
  }
  mean /= nb;
  *ghz = mean / (ns / nb);
  const double per_inst = (OP == MIX_ALU_FMA || OP == IMADWIDE || OP == ISETP_SEL) ? 2.0 : 1.0;
  const double thread_ops = (double)nb * 256 * ITER * CH * per_inst;
  // per SM-clock from the kernel's event time and the clock64/globaltimer SM clock (the blocks
  // need not all be co-resident, so per-block cycle counts would overstate the rate)
  return thread_ops / ((double)*ms * 1e-3 * (*ghz * 1e9) * sms);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, dev);
  const int bps = 4;
  int* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)sms * bps * 256 * sizeof(int));
  cudaMalloc(&cyc, (size_t)2 * sms * bps * sizeof(long long));
  long long* hcyc = (long long*)malloc((size_t)2 * sms * bps * sizeof(long long));
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_rate_khz\": %d, \"warps_per_sm\": %d, "
         "\"chains_per_thread\": %d, \"rates\": {\n", pr.name, sms, clk, bps * 8, CH);
  float ms;
  double v, ghz;
#define ONE(OPX, LAST)                                                                       \
  v = run<OPX>(sms, bps, out, cyc, hcyc, &ms, &ghz);                                         \
  printf("  \"%s\": {\"thread_ops_per_sm_clk\": %.2f, \"sm_clock_ghz\": %.3f, "            \
         "\"kernel_ms\": %.3f}%s\n", NAMES[OPX], v, ghz, ms, LAST ? "" : ",");
  ONE(IADD3, 0)
  ONE(LOP3, 0)
  ONE(IMAD, 0)
  ONE(ISETP_SEL, 0)
  ONE(IMADWIDE, 0)
  ONE(MIX_ALU_FMA, 0)
  ONE(LDS32, 0)
  ONE(SHFL, 0)
  ONE(VIMNMX, 1)
  printf("}}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
