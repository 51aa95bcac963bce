// Diagnostics with no reference counterpart: the measured tcgen05 kind::i8 dense
// peak of this device, the denominator of bench.py's roofline for the int8 conv
// kernel.  One CTA per SM, one warp issuing back-to-back M=128 x N=256 x K=32
// SS-mode MMAs (the shape that reaches the tensor floor, 128 cycles per MMA:
// profiles/mma_microbench2_r01.txt), operands resident in shared memory, one
// commit at the end; the host times the launch with CUDA events, so the number
// includes whatever SM clock the device holds under that load.
#include <cuda_runtime.h>

#include "abed_internal.h"
#include "ptx.cuh"

namespace abed_dev {

__global__ void __launch_bounds__(128, 1) mma_i8_peak_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t base = smem_u32(smem);
    const uint32_t idesc = make_idesc_i8(256);
    const uint64_t a = make_sdesc(base, 2048, 128);
    const uint64_t b = make_sdesc(base + 16 * 1024, 4096, 128);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) mma_i8_w(tmem, a + (j & 3) * 16, b + (j & 3) * 16, idesc, (it | j) ? 1u : 0u);
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace abed_dev

extern "C" int abed_probe_mma_i8_peak(int32_t iters, double* tops, double* ms) {
  using namespace abed_host;
  return guarded([&] {
    require_device();
    if (iters < 1) throw_invalid("probe: iters must be >= 1");
    const uint32_t smem = 48 * 1024;
    cuda_check(cudaFuncSetAttribute(abed_dev::mma_i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
               "probe attr");
    const int grid = num_sms();
    abed_dev::mma_i8_peak_kernel<<<grid, 128, smem>>>(iters / 8 > 0 ? iters / 8 : 1);  // warm-up
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    cuda_check(cudaEventRecord(e0), "record");
    abed_dev::mma_i8_peak_kernel<<<grid, 128, smem>>>(iters);
    cuda_check(cudaEventRecord(e1), "record");
    cuda_check(cudaEventSynchronize(e1), "probe sync");
    float t = 0.0f;
    cuda_check(cudaEventElapsedTime(&t, e0, e1), "elapsed");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double ops = 2.0 * 128 * 256 * 32 * 8.0 * iters * grid;
    *ms = t;
    *tops = ops / (t * 1e-3) / 1e12;
  });
}
