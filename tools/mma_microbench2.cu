// Microbenchmark 2: decides the conv mainloop orientation.
//   ss   : A,B from smem (A 128-B aligned or 16-B offset), kind::i8, M=128
//   ts   : A from TMEM, B from smem at 16-B offsets (the strip shift trick), N sweep
//   cp   : tcgen05.cp 128x256b smem -> TMEM alone (4 KB per copy)
//   tscp : one 4 KB tcgen05.cp (A ring refill) per TS MMA, N sweep
// One CTA per SM (148), operands resident, single issuing thread, clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_mb2 tools/mma_microbench2.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2006_04984_b200/csrc/ptx.cuh"

using namespace abed_dev;

// whole warp calls; one elected lane issues (no per-instruction ELECT loop)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_cp(uint32_t taddr, uint64_t sdesc) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void commit_e(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}

enum { SS_AL = 0, SS_OFF = 1, TS = 2, CP = 3, TSCP = 4, TSCP2 = 5 };

template <int mode>
__global__ void __launch_bounds__(128, 1) kern(int n, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t base = smem_u32(smem);
    const uint32_t idesc = make_idesc_i8(n);
    // B strip: 2 K-halves 4 KB apart (LBO), rows 16 B apart
    const uint64_t bstrip = make_sdesc(base + 100 * 1024, 4096, 128);
    const uint64_t aal = make_sdesc(base, 2048, 128);
    const uint64_t aoff = make_sdesc(base + 16, 2048, 128);
    uint32_t off[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) off[j] = ((j * 57 + 3) % 120);  // 16-B units (tap shifts)
    const uint32_t acc_cols = n;                                  // accumulator at col 0
    const uint32_t aring = tmem + ((acc_cols + 31) & ~31u);       // A ring after the acc
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t acc = (it | j) ? 1u : 0u;
        switch (mode) {
          case SS_AL: mma_ss(tmem, aal + (j & 3) * 256, bstrip + off[j], idesc, acc); break;
          case SS_OFF: mma_ss(tmem, aoff + off[j], bstrip + off[j], idesc, acc); break;
          case TS: mma_ts(tmem, aring + (j & 15) * 8, bstrip + off[j], idesc, acc); break;
          case CP: tc_cp(tmem + (j & 15) * 8, aal + (j & 3) * 256); break;
          case TSCP: {
            const uint32_t slot = aring + (j & 15) * 8;
            tc_cp(slot, aal + (j & 3) * 256);
            mma_ts(tmem, slot, bstrip + off[j], idesc, acc);
            break;
          }
          default: {  // TSCP2: one cp per two MMAs (A reused by two pixel tiles)
            const uint32_t slot = aring + (j >> 1) * 8;
            if ((j & 1) == 0) tc_cp(slot, aal + (j & 3) * 256);
            mma_ts(tmem, slot, bstrip + off[j], idesc, acc);
            break;
          }
        }
      }
    }
    commit_e(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  typedef void (*KF)(int, int, unsigned long long*);
  KF ks[6] = {kern<0>, kern<1>, kern<2>, kern<3>, kern<4>, kern<5>};
  for (auto k : ks) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"SS A-aligned", "SS A-offset", "TS", "CP only", "TS+cp/mma", "TS+cp/2mma"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int n : {16, 32, 48, 64, 96, 128, 160, 192, 256}) {
      if (mode == CP && n != 64) continue;
      const int iters = 256;
      ks[mode]<<<148, 128, 200 * 1024>>>(n, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("err %s (mode %d n %d)\n", cudaGetErrorString(e), mode, n);
        return 1;
      }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      const double per = avg / (iters * 16);
      if (mode == CP) {
        printf("%-12s        : %7.1f cyc/cp (4 KB) -> %.1f B/clk\n", names[mode], per, 4096.0 / per);
      } else {
        const double ideal = 128.0 * n / 256.0;
        printf("%-12s N=%3d : %7.1f cyc/mma (floor %5.1f) eff %.2f ; MAC/clk/SM %6.0f\n", names[mode], n, per, ideal,
               ideal / per, 128.0 * n * 32 / per);
      }
    }
  }
  return 0;
}
