// Microbenchmark: tcgen05.mma kind::i8 issue rate (cta_group::1, M=128) versus
// N and shared-memory operand layout (SWIZZLE_NONE aligned / 16-B offset start,
// SWIZZLE_128B).  One CTA per SM, operands resident in smem, no loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_mb tools/mma_microbench.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2006_04984_b200/csrc/ptx.cuh"

using namespace abed_dev;

__device__ uint64_t sdesc_sw128(uint32_t saddr) {
  // K-major SWIZZLE_128B: 8-row x 128-B atoms, SBO = 1024 B, LBO ignored (1)
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(128, 1) mb_kernel(int mode, int n, int iters, int per_commit, int chains, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tslot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t base = smem_u32(smem);
    const uint32_t idesc = make_idesc_i8(n);
    uint32_t phase = 0;
    const uint64_t a0 = make_sdesc(base + 16, 248 * 16, 128);
    const uint64_t b0 = make_sdesc(base + 100 * 1024, n * 16, 128);
    uint32_t aoff[18], boff[18];
#pragma unroll
    for (int j = 0; j < 18; ++j) { aoff[j] = (j * 57 + 3) & 1023; boff[j] = (j * 2 * n) & 2047; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 18; ++j) {
        if (chains == 1) mma_i8(tmem, a0 + aoff[j], b0 + boff[j], idesc, (it | j) ? 1u : 0u);
        else mma_i8(tmem + (j & 1) * n, a0 + aoff[j], b0 + boff[j], idesc, (it | (j >> 1)) ? 1u : 0u);
      }
      if (per_commit == 1) { mma_commit(&bar); mbar_wait(&bar, phase); phase ^= 1; }
    }
    if (per_commit != 1) { mma_commit(&bar); mbar_wait(&bar, 0); }
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__global__ void __launch_bounds__(128, 1) ts_kernel(int n, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tslot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t base = smem_u32(smem);
    const uint32_t idesc = make_idesc_i8(n);
    const uint64_t b0 = make_sdesc(base + 16, 248 * 16, 128);
    uint32_t boff[18], aoff[18];
#pragma unroll
    for (int j = 0; j < 18; ++j) { boff[j] = (j * 57 + 3) & 1023; aoff[j] = 256 + (j % 16) * 8; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 18; ++j) mma_i8_ts(tmem, tmem + aoff[j], b0 + boff[j], idesc, (it | j) ? 1u : 0u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(mb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"none-aligned", "none-offset", "sw128"};
  for (int mode : {1})
    for (int n : {64, 128, 256})
      for (int chains : {1})
      for (int pc : {0}) {
        if (chains * n > 512) continue;
        const int iters = 200;
        mb_kernel<<<148, 128, 200 * 1024>>>(mode, n, iters, pc, chains, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double per = avg / (iters * 18);
        const double ideal = 128.0 * n / 256.0;
        printf("%-13s N=%3d chains=%d pc=%2d : %7.1f cyc/mma (ideal %5.1f) -> %5.2fx ; MAC/cyc/SM %6.0f\n", names[mode], n, chains, pc,
               per, ideal, per / ideal, 128.0 * n * 32 / per);
      }
  cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {64, 128, 256}) {
    if (n > 256) continue;
    const int iters = 200;
    ts_kernel<<<148, 128, 200 * 1024>>>(n, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double per = avg / (iters * 18);
    printf("TS (A in TMEM) N=%3d : %7.1f cyc/mma (ideal %5.1f) ; MAC/cyc/SM %6.0f\n", n, per, 128.0 * n / 256.0, 128.0 * n * 32 / per);
  }
  return 0;
}
