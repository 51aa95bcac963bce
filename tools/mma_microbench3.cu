// Microbenchmark 3: the conv kernel's MMA issue pattern in isolation.
// Layer-1 geometry (C=K=64, 3x3, Wl=57, strip 248 px, 4 channel groups per
// stage), B resident, A strips in a 4-stage ring, two alternating TMEM
// accumulators, one commit per unit; optional concurrent bulk copies into the
// A ring (the producer's traffic) and a waiting "epilogue" warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_mb3 tools/mma_microbench3.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2006_04984_b200/csrc/ptx.cuh"

using namespace abed_dev;

constexpr int kStrip = 248, kGps = 4, kStages = 4, kUnits = 64;
constexpr uint32_t kStripBytes = kStrip * 16, kAStage = kGps * kStripBytes;

// SPIN: warps >= 2 spin on mbarrier.try_wait of the "done" barrier (like idle epilogue warps)
__device__ int g_fill = 0;  // 0: i*2654435761, 1: zeros, 2: SplitMix64 random bytes, 3: all 0x7f
template <int N, bool COPIES, bool SPIN>
__global__ void __launch_bounds__(384, 1) kern(const int8_t* gsrc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_done, bar_copy, bar_final;
  __shared__ uint32_t tslot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
    uint32_t v = i * 2654435761u;
    if (g_fill == 1) v = 0u;
    if (g_fill == 2) {
      uint64_t z = (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull + blockIdx.x;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      v = (uint32_t)(z ^ (z >> 31));
    }
    if (g_fill == 3) v = 0x7f7f7f7fu;
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar_done, 1);
    mbar_init(&bar_copy, 1);
    mbar_init(&bar_final, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kAStage;
  if (warp == 0) {
    const uint32_t idesc = make_idesc_i8(N);
    long long t0 = clock64();
    for (int u = 0; u < kUnits; ++u) {
      const int stage = u % kStages;
      const uint64_t a0 = make_sdesc(smem_u32(sA + stage * kAStage), kStripBytes, 128u);
      const uint64_t b0 = make_sdesc(smem_u32(sB), N * 16u, 128u);
      const uint32_t a_lo = static_cast<uint32_t>(a0), a_hi = static_cast<uint32_t>(a0 >> 32);
      const uint32_t b_lo = static_cast<uint32_t>(b0), b_hi = static_cast<uint32_t>(b0 >> 32);
      const uint32_t d = tmem + (u & 1) * N;
      uint32_t acc = 0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
          for (int g = 0; g < kGps; g += 2) {
            const uint32_t ao = a_lo + (r * 57 + s) + g * kStrip;
            const uint32_t bo = b_lo + ((r * 3 + s) * kGps + g) * N;
            mma_i8_w(d, (static_cast<uint64_t>(a_hi) << 32) | ao, (static_cast<uint64_t>(b_hi) << 32) | bo, idesc, acc);
            acc = 1;
          }
      mma_commit_w(&bar_done);
    }
    mma_commit_w(&bar_final);  // arrives once every MMA above has completed
    mbar_wait(&bar_final, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (SPIN && warp >= 2) {
    mbar_wait(&bar_final, 0);
  } else if (COPIES && warp == 1) {
    // the producer's traffic: one A stage (4 strips) per unit into the ring
    for (int u = 0; u < kUnits; ++u) {
      const int stage = (u + 2) % kStages;
      mbar_arrive_expect_tx_w(&bar_copy, kAStage);
      for (int g = 0; g < kGps; ++g)
        bulk_g2s_w(sA + stage * kAStage + g * kStripBytes, gsrc + (static_cast<int64_t>(blockIdx.x) * kUnits + u) * kAStage + g * kStripBytes,
                   kStripBytes, &bar_copy);
      mbar_wait(&bar_copy, u & 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// the conv kernel's loop: runtime R, S, strides, gps, Wl, strip (uniform counters)
struct Geo { int R, S, sh, sw, nph_w, gps, Wl, strip, n, units, k_stages; };
__global__ void __launch_bounds__(128, 1) kern_rt(const __grid_constant__ Geo q, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_done, bar_final;
  __shared__ uint32_t tslot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(&bar_done, 1);
    mbar_init(&bar_final, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  uint8_t* sA = smem;
  const uint32_t a_stage = q.gps * q.strip * 16;
  uint8_t* sB = smem + kStages * a_stage;
  if (warp == 0) {
    const uint32_t idesc = make_idesc_i8(q.n);
    const uint32_t strip16 = q.strip, blbo16 = q.n;
    long long t0 = clock64();
    int stage = 0;
    for (int u = 0; u < q.units; ++u) {
      const uint32_t d = tmem + (u & 1) * q.n;
      for (int ks = 0; ks < q.k_stages; ++ks) {
        const uint64_t a0 = make_sdesc(smem_u32(sA + stage * a_stage), q.strip * 16u, 128u);
        const uint64_t b0 = make_sdesc(smem_u32(sB), q.n * 16u, 128u);
        uint32_t accum = ks > 0 ? 1u : 0u;
        const uint32_t a_lo = static_cast<uint32_t>(a0), a_hi = static_cast<uint32_t>(a0 >> 32);
        const uint32_t b_lo = static_cast<uint32_t>(b0), b_hi = static_cast<uint32_t>(b0 >> 32);
        const uint32_t ph_row = static_cast<uint32_t>(q.nph_w * q.gps) * strip16;
        const uint32_t ph_col = static_cast<uint32_t>(q.gps) * strip16;
        uint32_t bo = b_lo;
        uint32_t r_ph = 0, r_q = 0;
        for (int r = 0; r < q.R; ++r) {
          const uint32_t roff = a_lo + r_ph * ph_row + r_q * static_cast<uint32_t>(q.Wl);
          uint32_t s_ph = 0, s_q = 0;
          for (int sc = 0; sc < q.S; ++sc) {
            const uint32_t ao = roff + s_ph * ph_col + s_q;
#pragma unroll 2
            for (int g = 0; g < q.gps; g += 2) {
              const uint64_t ad = (static_cast<uint64_t>(a_hi) << 32) | (ao + g * strip16);
              const uint64_t bd = (static_cast<uint64_t>(b_hi) << 32) | (bo + g * blbo16);
              mma_i8_w(d, ad, bd, idesc, accum);
              accum = 1u;
            }
            bo += static_cast<uint32_t>(q.gps) * blbo16;
            if (++s_ph == static_cast<uint32_t>(q.sw)) { s_ph = 0; ++s_q; }
          }
          if (++r_ph == static_cast<uint32_t>(q.sh)) { r_ph = 0; ++r_q; }
        }
        mma_commit_w(&bar_done);
        if (++stage == kStages) stage = 0;
      }
    }
    mma_commit_w(&bar_final);
    mbar_wait(&bar_final, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

void run_rt(const char* name, Geo g, unsigned long long* d) {
  cudaFuncSetAttribute(kern_rt, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  kern_rt<<<148, 128, 200 * 1024>>>(g, d);
  kern_rt<<<148, 128, 200 * 1024>>>(g, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const int mmas = g.units * g.k_stages * g.R * g.S * (g.gps / 2);
  printf("%-28s N=%3d : %6.1f cyc/mma (%d MMAs)\n", name, g.n, avg / mmas, mmas);
}

template <int N, bool C, bool SPIN = false>
void run(const char* name, const int8_t* src, unsigned long long* d, int threads = 128) {
  cudaFuncSetAttribute(kern<N, C, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  kern<N, C, SPIN><<<148, threads, 200 * 1024>>>(src, d);
  kern<N, C, SPIN><<<148, threads, 200 * 1024>>>(src, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("err %s\n", cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / (kUnits * 18);
  printf("%-28s N=%3d : %6.1f cyc/mma (floor %5.1f, smem model %5.1f)\n", name, N, per, N / 2.0,
         (4096.0 + 32 * N + (C ? kAStage / 18.0 : 0)) / 128.0);
}

int main() {
  unsigned long long* d;
  int8_t* src;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&src, (size_t)148 * kUnits * kAStage);
  cudaMemset(src, 1, (size_t)148 * kUnits * kAStage);
  run<64, false>("L1 pattern, no copies", src, d);
  run<64, true>("L1 pattern, + bulk copies", src, d);
  run<80, false>("L1 pattern (FC), no copies", src, d);
  run<128, false>("L1 pattern N=128", src, d);
  run<128, true>("L1 pattern N=128 + copies", src, d);
  for (int f = 0; f < 4; ++f) {
    cudaMemcpyToSymbol(g_fill, &f, sizeof(int));
    const char* nm[] = {"fill i*golden", "fill zeros", "fill splitmix random", "fill all 0x7f"};
    run<64, false>(nm[f], src, d);
    run<128, false>(nm[f], src, d);
  }
  int z = 0;
  cudaMemcpyToSymbol(g_fill, &z, sizeof(int));
  run_rt("runtime loop L1 (6 units)", Geo{3, 3, 1, 1, 1, 4, 57, 248, 64, 6, 1}, d);
  run_rt("runtime loop L1 (64 units)", Geo{3, 3, 1, 1, 1, 4, 57, 248, 64, 64, 1}, d);
  run_rt("runtime loop L4 (8 stages)", Geo{3, 3, 1, 1, 1, 4, 8, 152, 64, 1, 8}, d);
  run_rt("runtime loop L2 N=128", Geo{3, 3, 1, 1, 1, 4, 29, 192, 128, 2, 2}, d);
  run<64, false>("384 thr, idle warps", src, d, 384);
  run<64, false, true>("384 thr, 10 warps try_wait", src, d, 384);
  run<64, true, true>("384 thr, spin + copies", src, d, 384);
  return 0;
}
