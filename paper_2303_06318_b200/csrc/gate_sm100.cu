// gate_sm100.cu -- the top-1 gate (gate_forward, moe.cpp:158-186) on the 5th-gen tensor
// cores: logits = a Wg for 128-token tiles as tcgen05.mma M128 x N(E') x K16, the token rows
// and the transposed gate weight streamed by TMA through an mbarrier ring (the gate reads
// every token row once: it is HBM-bound, and TMA keeps the whole stream in flight without
// register or thread cost), fp32 accumulators in TMEM (double-buffered across tiles), and an
// epilogue in which each thread owns one token: its E logits come out of TMEM into registers,
// the argmax scans them exactly like the reference (strict >, ascending j: lowest index wins
// ties, NaN never wins except at j = 0) and the softmax subtracts the top logit.
// Persistent CTAs; warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 = TMEM allocator,
// warps 4-7 = epilogue (warp w owns TMEM lanes / tokens 32*(w%4)..+31 of the tile).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ted_internal.h"
#include "ted_ptx.cuh"

namespace ted {
namespace {

constexpr int GBM = 128, GBK = 64, GSTAGES = 6;
// K-block kb accumulates into partial kb % NACC: with N = E' <= 64 a tcgen05.mma is tiny and
// one accumulator would serialise the whole K loop on the MMA latency; NACC independent
// chains keep the tensor core fed, the epilogue sums them in a fixed order (deterministic,
// identical on every TP replica)
constexpr int NACC = 4;

template <int EP>
struct GateCfg {
  static constexpr int A_BYTES = GBM * GBK * 2;  // 16 KB
  static constexpr int B_BYTES = EP * GBK * 2;   // 2-8 KB
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr uint32_t TCOLS = 2 * NACC * EP;  // two buffers of NACC partials (128-512)
  static constexpr size_t BAR_OFF = size_t(GSTAGES) * STAGE;
  static constexpr size_t SMEM = 1024 + BAR_OFF + 256 + 2 * 64 * sizeof(int);
};

__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int EP>
__global__ void __launch_bounds__(256, 1)
    gate_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int64_t n, int h, int E, float* __restrict__ logits, float* __restrict__ probs,
                   int* __restrict__ expert, float* __restrict__ prob, int* __restrict__ blk_hist) {
  using CF = GateCfg<EP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::BAR_OFF);
  uint64_t* empty = full + GSTAGES;
  uint64_t* tfull = empty + GSTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_hist = reinterpret_cast<int*>(smem + CF::BAR_OFF + 256);  // [2 blocks][64]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = int((n + GBM - 1) / GBM);
  const int kb_n = h / GBK;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int st = 0; st < GSTAGES; ++st) {
      ptx::mbar_init(&full[st], 1);
      ptx::mbar_init(&empty[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4);  // the four epilogue warps
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(s_tmem, CF::TCOLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < kb_n; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (ptx::elect_one()) {
          uint8_t* st = smem + size_t(stage) * CF::STAGE;
          ptx::mbar_arrive_expect_tx(&full[stage], CF::STAGE);
          ptx::tma_load_3d(st, &tmA, &full[stage], kb * GBK, t * GBM, 0);
          ptx::tma_load_3d(st + CF::A_BYTES, &tmB, &full[stage], kb * GBK, 0, 0);
        }
        __syncwarp();
        if (++stage == GSTAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = ptx::idesc_bf16(GBM, EP, false, false);
    const uint32_t base = ptx::smem_u32(smem);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t tmem_d0 = tmem_base + acc * (NACC * EP);
      for (int kb = 0; kb < kb_n; ++kb) {
        const uint32_t tmem_d = tmem_d0 + (kb % NACC) * EP;
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t sa = base + stage * CF::STAGE;
        const uint64_t ad = ptx::sdesc_sw128(sa, 16, 1024);
        const uint64_t bd = ptx::sdesc_sw128(sa + CF::A_BYTES, 16, 1024);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k)
            ptx::umma_bf16(tmem_d, ad + k * 2, bd + k * 2, idesc, (kb / NACC | k) != 0);
          ptx::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == GSTAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue: one token per thread
    const int et = threadIdx.x - 128;  // 0..127 = token row of the tile
    const int sp = warp & 3;
    const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      s_hist[et] = 0;  // [2][64]: the tile's two 64-token routing blocks
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      float l[EP];
      const uint32_t ta = tmem_base + acc * (NACC * EP) + (uint32_t(sp * 32) << 16);
#pragma unroll
      for (int j = 0; j < EP; ++j) l[j] = 0.f;
#pragma unroll
      for (int q = 0; q < NACC; ++q) {  // partials of K-blocks q, q + NACC, ... (kb_n >= NACC)
        if (q >= kb_n) break;
        if constexpr (EP == 16) {
          float v[16];
          ptx::tmem_ld16(ta + q * EP, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) l[i] += v[i];
        } else {
#pragma unroll
          for (int c = 0; c < EP; c += 32) {
            float v[32];
            ptx::tmem_ld32(ta + q * EP + c, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) l[c + i] += v[i];
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      named_sync(1, 128);  // s_hist zeroed
      const int64_t k = int64_t(t) * GBM + et;
      if (k < n) {
        // argmax exactly as moe.cpp:166-174 (top = l[0]; strict > over ascending j)
        int best = 0;
        float top = l[0];
#pragma unroll
        for (int j = 1; j < EP; ++j)
          if (j < E && l[j] > top) {
            top = l[j];
            best = j;
          }
        const float mx = isnan(l[0]) ? l[0] : top;
        float e[EP], sum = 0.f;
#pragma unroll
        for (int j = 0; j < EP; ++j) {
          e[j] = j < E ? expf(l[j] - mx) : 0.f;
          sum += e[j];
        }
        float* lrow = logits ? logits + k * E : nullptr;
        float* prow = probs + k * E;
        float pb = 0.f;
#pragma unroll
        for (int j = 0; j < EP; ++j) {
          if (j >= E) break;
          const float pj = e[j] / sum;
          prow[j] = pj;
          if (lrow) lrow[j] = l[j];
          if (j == best) pb = pj;
        }
        expert[k] = best;
        prob[k] = pb;
        atomicAdd(&s_hist[(et >> 6) * 64 + best], 1);
      }
      named_sync(1, 128);
      const int b = t * 2 + (et >> 6), e2 = et & 63;
      if (e2 < E && b < nblk) blk_hist[int64_t(b) * E + e2] = s_hist[et];
      named_sync(1, 128);  // s_hist read before the next tile zeroes it
    }
  }
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, CF::TCOLS);
}

template <int EP>
cudaError_t launch_gate(const CUtensorMap& ma, const CUtensorMap& mb, int64_t n, int h, int E,
                        float* logits, float* probs, int* expert, float* prob, int* blk_hist,
                        cudaStream_t s) {
  auto k = gate_tc_kernel<EP>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(GateCfg<EP>::SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int ntiles = int((n + GBM - 1) / GBM);
  const int grid = ntiles < sm_count() ? ntiles : sm_count();
  k<<<grid, 256, GateCfg<EP>::SMEM, s>>>(ma, mb, n, h, E, logits, probs, expert, prob, blk_hist);
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace

int gate_tc_experts(int E) { return E <= 16 ? 16 : (E <= 32 ? 32 : 64); }

// a [n][h] bf16, wgT [EP][h] bf16 (the transposed gate weight, zero rows e >= E)
cudaError_t gate_forward_tc(const bf16* a, const bf16* wgT, int64_t n, int h, int E,
                            float* logits, float* probs, int* expert, float* prob,
                            int* blk_hist, cudaStream_t s) {
  if (E < 1 || E > 64 || h % GBK != 0 || n < 1 || n > INT32_MAX) return cudaErrorInvalidValue;
  const int EP = gate_tc_experts(E);
  CUtensorMap ma, mb;
  if (!tmap_bf16_2d(&ma, a, uint64_t(h), uint64_t(n), uint64_t(h) * 2, GBK, GBM) ||
      !tmap_bf16_2d(&mb, wgT, uint64_t(h), uint64_t(EP), uint64_t(h) * 2, GBK, uint32_t(EP)))
    return cudaErrorInvalidValue;
  if (EP == 16) return launch_gate<16>(ma, mb, n, h, E, logits, probs, expert, prob, blk_hist, s);
  if (EP == 32) return launch_gate<32>(ma, mb, n, h, E, logits, probs, expert, prob, blk_hist, s);
  return launch_gate<64>(ma, mb, n, h, E, logits, probs, expert, prob, blk_hist, s);
}

}  // namespace ted
