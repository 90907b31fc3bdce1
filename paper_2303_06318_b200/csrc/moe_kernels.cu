// moe_kernels.cu -- HBM-bound kernels of the TED MoE layer on sm_100a:
//   gate: argmax + softmax on given logits (the logits themselves: gate_sm100.cu) moe.cpp:158-186
//   capacity slot scan (exclusive per-expert prefix, ascending)     moe.cpp:454-462 order
//   dispatch pack (DTD chunk select + scatter into expert layout)   moe.cpp:440-476
//   combine y = p * f_home, and its backward                        moe.cpp:558-563, :587-597
//   gate backward (dlogits, dWg = a^T dl, da += dl Wg^T)            moe.cpp:188-208, :685
//   per-expert bias-gradient column sums                            nn.cpp:70-76
//   tiled AdamW                                                     optimizer.cpp:58-104
// Design: 64-token routing blocks (16K tokens -> 256 CTAs, > 148 SMs), one warp per 8
// tokens, every row access a 16-byte vector with several loads in flight per lane
// (two token rows interleaved), all reductions deterministic (fixed order, no float
// atomics).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <atomic>

#include "ted_internal.h"
#include "ted_vec.cuh"

namespace ted {

std::atomic<unsigned long long> g_launches{0};
unsigned long long launches() { return g_launches.load(); }
void count_launch(int k) { g_launches += k; }

namespace {

constexpr int kThreads = 256;              // 8 warps
constexpr int kWarpTok = kRouteBlock / 8;  // tokens per warp (8)

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------------ gate forward
// Candidate order for top-1: strictly larger value wins, equal values -> lower index.
// NaN logits at j > 0 never win; a NaN at j = 0 pins the choice to expert 0 (the
// reference scans `if (l[j] > top)` from top = l[0], moe.cpp:167-174).
__device__ __forceinline__ bool cand_better(float va, int ia, float vb, int ib) {
  if (ib < 0) return false;
  if (ia < 0) return true;
  return (vb > va) || (vb == va && ib < ia);
}

// Per-token selection + softmax; the token's E logits are spread over the warp (lane l
// holds j = l and j = l + 32).  Writes outputs; returns best (all lanes).
__device__ __forceinline__ int select_softmax(float l0v, float l1v, int E, int lane, int64_t k,
                                              float* logits, float* probs, int* expert,
                                              float* prob) {
  const int j0 = lane, j1 = lane + 32;
  const bool ok0 = j0 < E, ok1 = j1 < E;
  float bv = 0.f;
  int bi = -1;
  if (ok0 && !isnan(l0v)) { bv = l0v; bi = j0; }
  if (ok1 && !isnan(l1v) && cand_better(bv, bi, l1v, j1)) { bv = l1v; bi = j1; }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(FULL, bv, o);
    const int oi = __shfl_xor_sync(FULL, bi, o);
    if (cand_better(bv, bi, ov, oi)) { bv = ov; bi = oi; }
  }
  const float first = __shfl_sync(FULL, l0v, 0);
  if (isnan(first) || bi < 0) bi = 0;
  const float top = isnan(first) ? first : bv;
  const float e0 = ok0 ? expf(l0v - top) : 0.f;
  const float e1 = ok1 ? expf(l1v - top) : 0.f;
  const float sum = warp_sum(e0 + e1);
  const float p0 = e0 / sum, p1 = e1 / sum;
  if (ok0) {
    probs[k * E + j0] = p0;
    if (logits) logits[k * E + j0] = l0v;
  }
  if (ok1) {
    probs[k * E + j1] = p1;
    if (logits) logits[k * E + j1] = l1v;
  }
  const float pb = __shfl_sync(FULL, bi < 32 ? p0 : p1, bi & 31);
  if (lane == 0) {
    expert[k] = bi;
    prob[k] = pb;
  }
  return bi;
}

// Stage Wg[c0:c0+hc, :] transposed into smem as [EMAX][HC] bf16 (zero for j >= E).
template <int EMAX>
__device__ __forceinline__ void stage_wg(const bf16* __restrict__ wg, int E, int c0, int hc,
                                         int HC, bf16* s_wg) {
  if (E % 8 == 0) {
    // rows of Wg are E contiguous bf16: one 16 B vector per 8 experts, coalesced
    const int vpr = E / 8;
    for (int idx = threadIdx.x; idx < hc * vpr; idx += blockDim.x) {
      const int i = idx / vpr, q = idx % vpr;
      const uint4 u = *reinterpret_cast<const uint4*>(wg + int64_t(c0 + i) * E + q * 8);
      const bf16* pv = reinterpret_cast<const bf16*>(&u);
#pragma unroll
      for (int j = 0; j < 8; ++j) s_wg[(q * 8 + j) * HC + i] = pv[j];
    }
    for (int idx = threadIdx.x; idx < (EMAX - E) * hc; idx += blockDim.x)
      s_wg[(E + idx / hc) * HC + idx % hc] = __float2bfloat16(0.f);
  } else {
    for (int idx = threadIdx.x; idx < EMAX * hc; idx += blockDim.x) {
      const int j = idx / hc, i = idx % hc;
      s_wg[j * HC + i] = j < E ? wg[int64_t(c0 + i) * E + j] : __float2bfloat16(0.f);
    }
  }
}

// mma.sync.m16n8k16 (bf16 in, fp32 accumulate): the gate backward's small products
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1,
                                               uint32_t a2, uint32_t a3, uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// wgT[e][k] = Wg[k][e] (e < E), 0 (E <= e < EMAX)
__global__ void wg_transpose_kernel(const bf16* __restrict__ wg, int h, int E, int EMAX,
                                    bf16* __restrict__ wgT) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= h) return;
  for (int e = 0; e < EMAX; ++e)
    wgT[int64_t(e) * h + k] = e < E ? wg[int64_t(k) * E + e] : __float2bfloat16(0.f);
}

__global__ void __launch_bounds__(kThreads) route_logits_kernel(const float* __restrict__ L,
                                                                int64_t n, int E,
                                                                float* __restrict__ probs,
                                                                int* __restrict__ expert,
                                                                float* __restrict__ prob,
                                                                int* __restrict__ blk_hist) {
  __shared__ int s_hist[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 64) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock;
  for (int t = 0; t < kWarpTok; ++t) {
    const int64_t k = tok0 + warp * kWarpTok + t;
    if (k >= n) break;
    const float l0v = lane < E ? L[k * E + lane] : 0.f;
    const float l1v = lane + 32 < E ? L[k * E + lane + 32] : 0.f;
    const int best = select_softmax(l0v, l1v, E, lane, k, nullptr, probs, expert, prob);
    if (lane == 0) atomicAdd(&s_hist[best], 1);
  }
  __syncthreads();
  if (threadIdx.x < E) blk_hist[int64_t(blockIdx.x) * E + threadIdx.x] = s_hist[threadIdx.x];
}

// ------------------------------------------------------------------ route scan (1 CTA)
// Thread (e, p) owns a contiguous range of blocks for expert e: range sums, an exclusive
// scan over the ranges, then the per-block exclusive prefixes.
__global__ void __launch_bounds__(kThreads) route_scan_kernel(RouteScanArgs A) {
  const int E = A.E, T = A.T;
  const int64_t n = A.n;
  const int nblk = int((n + kRouteBlock - 1) / kRouteBlock);
  __shared__ int s_rng[kThreads];
  __shared__ int s_S[9 * 64];   // [(T+1)][E]
  __shared__ int s_kc[8 * 64];  // [T][E]
  const int parts = kThreads / E;  // >= 4 (E <= 64)
  const int chunk = (nblk + parts - 1) / parts;
  const int tid = threadIdx.x;
  const int e = tid % E, p = tid / E;
  const bool active = p < parts;
  const int b0 = p * chunk, b1 = min(nblk, b0 + chunk);
  int sum = 0;
  if (active)
    for (int b = b0; b < b1; ++b) sum += A.blk_hist[int64_t(b) * E + e];
  s_rng[tid] = sum;
  __syncthreads();
  if (tid < E) {  // exclusive scan over parts for expert tid
    int acc = 0;
    for (int q = 0; q < parts; ++q) {
      const int v = s_rng[q * E + tid];
      s_rng[q * E + tid] = acc;
      acc += v;
    }
    s_S[T * E + tid] = acc;  // boundary c = T: all tokens
  }
  __syncthreads();
  if (active) {
    int acc = s_rng[tid];
    for (int b = b0; b < b1; ++b) {
      A.blk_prefix[int64_t(b) * E + e] = acc;
      acc += A.blk_hist[int64_t(b) * E + e];
    }
  }
  __syncthreads();
  // per-expert token count before each chunk boundary c * n/T (c < T)
  for (int idx = tid; idx < T * E; idx += blockDim.x) {
    const int c = idx / E, ee = idx % E;
    const int64_t B = (n / T) * c;
    const int64_t bb = B / kRouteBlock;
    int acc;
    if (bb < nblk) {
      acc = A.blk_prefix[bb * E + ee];
      for (int64_t k = bb * kRouteBlock; k < B; ++k) acc += (A.expert[k] == ee);
    } else {
      acc = s_S[T * E + ee];
    }
    s_S[c * E + ee] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < (T + 1) * E; idx += blockDim.x) A.chunk_prefix[idx] = s_S[idx];
  for (int idx = tid; idx < T * E; idx += blockDim.x) {
    const int c = idx / E, ee = idx % E;
    const int64_t hi = lmin(A.cap, s_S[(c + 1) * E + ee]);
    const int64_t lo = lmin(A.cap, s_S[c * E + ee]);
    s_kc[idx] = int(hi - lo);
    A.kc[idx] = int(hi - lo);
  }
  __syncthreads();
  if (tid == 0) {
    if (A.local) {
      int off = 0;
      for (int ee = 0; ee < E; ++ee) {
        A.seg_off[ee] = off;
        A.send_base[ee] = off;
        A.home_base[ee] = off;
        off += (s_kc[ee] + kPad - 1) / kPad * kPad;
      }
      A.seg_off[E] = off;
    } else {
      int blockbase = 0;
      for (int c = 0; c < T; ++c) {
        int off = 0;
        for (int ee = 0; ee < E; ++ee) {
          A.home_base[c * E + ee] = blockbase + off;
          if (c == (A.my_chunk < 0 ? 0 : A.my_chunk)) A.send_base[ee] = off;
          off += s_kc[c * E + ee];
        }
        blockbase += off;
      }
    }
  }
}

// ------------------------------------------------------------------ row movers
// Copy rows with U 16-byte loads in flight per lane per row, two rows interleaved.
template <int U>
__device__ __forceinline__ void copy_rows2(const bf16* s0, bf16* d0, const bf16* s1, bf16* d1,
                                           int vec, int lane) {
  for (int base = lane; base < vec; base += 32 * U) {
    uint4 v0[U], v1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * 32;
      if (i < vec) {
        if (s0) v0[u] = ldg_stream(reinterpret_cast<const uint4*>(s0) + i);
        if (s1) v1[u] = ldg_stream(reinterpret_cast<const uint4*>(s1) + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * 32;
      if (i < vec) {
        if (s0) reinterpret_cast<uint4*>(d0)[i] = v0[u];
        if (s1) reinterpret_cast<uint4*>(d1)[i] = v1[u];
      }
    }
  }
}

// ------------------------------------------------------------------ dispatch
__global__ void __launch_bounds__(kThreads) dispatch_kernel(
    const bf16* __restrict__ a, int64_t n, int h, int E, int T, int my_chunk, int64_t cap,
    const int* __restrict__ expert, const int* __restrict__ blk_prefix,
    const int* __restrict__ chunk_prefix, const int* __restrict__ send_base,
    const int* __restrict__ home_base, int* __restrict__ slot_out, int* __restrict__ pos_send,
    int* __restrict__ pos_home, bf16* __restrict__ xsend) {
  __shared__ int s_wcnt[kRouteBlock / 32][64];
  __shared__ int s_pos[kRouteBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (kRouteBlock / 32) * 64; i += blockDim.x) (&s_wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t k = int64_t(blockIdx.x) * kRouteBlock + threadIdx.x;
  const bool ranker = threadIdx.x < kRouteBlock;  // warp-uniform (kRouteBlock % 32 == 0)
  const bool valid = ranker && k < n;
  const int e = valid ? expert[k] : -1;
  int rank = 0;
  if (ranker) {
    const unsigned mask = __match_any_sync(FULL, e);
    rank = __popc(mask & ((1u << lane) - 1u));
    if (valid && rank == 0) s_wcnt[warp][e] = __popc(mask);
  }
  __syncthreads();
  if (ranker) {
    int ps = -1;
    if (valid) {
      int pre = 0;
      for (int w = 0; w < warp; ++w) pre += s_wcnt[w][e];
      const int64_t slot = int64_t(blk_prefix[int64_t(blockIdx.x) * E + e]) + pre + rank;
      if (slot_out) slot_out[k] = int(slot);
      int c = 0;
      if (T > 1) {
        c = int(k / (n / T));
        if (c >= T) c = T - 1;
      }
      int ph = -1;
      if (slot < cap) {
        const int64_t before = lmin(cap, chunk_prefix[c * E + e]);
        const int r = int(slot - before);
        ph = home_base[c * E + e] + r;
        if (my_chunk < 0 || c == my_chunk) ps = send_base[e] + r;
      }
      pos_home[k] = ph;
      pos_send[k] = ps;
    }
    s_pos[threadIdx.x] = ps;
  }
  __syncthreads();
  if (xsend == nullptr || h == 0) return;
  const int vec = h / 8;
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock;
  for (int t = warp * kWarpTok; t < warp * kWarpTok + kWarpTok; t += 2) {
    const int p0 = s_pos[t], p1 = s_pos[t + 1];
    copy_rows2<4>(p0 >= 0 ? a + (tok0 + t) * h : nullptr, xsend + int64_t(p0 < 0 ? 0 : p0) * h,
                  p1 >= 0 ? a + (tok0 + t + 1) * h : nullptr,
                  xsend + int64_t(p1 < 0 ? 0 : p1) * h, vec, lane);
  }
}

__global__ void zero_pad_kernel(bf16* buf, int64_t ld, int h, const int* seg_off,
                                const int* valid, int G) {
  const int g = blockIdx.y;
  const int64_t r0 = int64_t(seg_off[g]) + valid[g];
  const int64_t r1 = seg_off[g + 1];
  const int vec = h / 8;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int64_t r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
    uint4* dst = reinterpret_cast<uint4*>(buf + r * ld);
    for (int i = threadIdx.x; i < vec; i += blockDim.x) dst[i] = z;
  }
}

// ------------------------------------------------------------------ combine
__global__ void __launch_bounds__(kThreads, 4) combine_fwd_kernel(const bf16* __restrict__ fhome,
                                                               const int* __restrict__ pos_home,
                                                               const float* __restrict__ prob,
                                                               int64_t n, int h,
                                                               bf16* __restrict__ y,
                                                               float* __restrict__ loss_part) {
  __shared__ float s_red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = h / 8;
  float sq = 0.f;
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock + warp * kWarpTok;
  for (int t = 0; t < kWarpTok; t += 2) {
    const int64_t k0 = tok0 + t, k1 = tok0 + t + 1;
    const bool v0 = k0 < n, v1 = k1 < n;
    const int p0 = v0 ? pos_home[k0] : -1, p1 = v1 ? pos_home[k1] : -1;
    const float q0 = v0 ? prob[k0] : 0.f, q1 = v1 ? prob[k1] : 0.f;
    for (int base = lane; base < vec; base += 32 * 4) {
      uint4 f0[4], f1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        f0[u] = make_uint4(0, 0, 0, 0);
        f1[u] = make_uint4(0, 0, 0, 0);
        if (i < vec) {
          if (p0 >= 0) f0[u] = ldg_stream(fhome + int64_t(p0) * h + i * 8);
          if (p1 >= 0) f1[u] = ldg_stream(fhome + int64_t(p1) * h + i * 8);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        if (i >= vec) continue;
        float f[8];
        if (v0) {
          unpack8(f0[u], f);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            f[q] *= q0;
            sq = fmaf(f[q], f[q], sq);
          }
          reinterpret_cast<uint4*>(y + k0 * h)[i] = pack8(f);
        }
        if (v1) {
          unpack8(f1[u], f);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            f[q] *= q1;
            sq = fmaf(f[q], f[q], sq);
          }
          reinterpret_cast<uint4*>(y + k1 * h)[i] = pack8(f);
        }
      }
    }
  }
  sq = warp_sum(sq);
  if (lane == 0) s_red[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0 && loss_part) {
    float tot = 0.f;
    for (int w = 0; w < 8; ++w) tot += s_red[w];
    loss_part[blockIdx.x] = tot;
  }
}

__global__ void loss_finalize_kernel(const float* part, int nblk, double inv_2n, double* loss) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) acc += part[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = s[0] * inv_2n;
}

// dfe[pos_send] = p * dy; dchosen = <f_home, dy>; dlogits = dchosen p_e (delta - p_j)
__global__ void __launch_bounds__(kThreads) combine_bwd_kernel(
    const bf16* __restrict__ fhome, const int* __restrict__ pos_home,
    const int* __restrict__ pos_send, const float* __restrict__ prob,
    const float* __restrict__ probs, const int* __restrict__ expert, int64_t n, int h, int E,
    const bf16* __restrict__ dy, const bf16* __restrict__ y, float dy_scale,
    bf16* __restrict__ dfe, float* __restrict__ dlogits) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = h / 8;
  const bf16* dsrc_base = dy ? dy : y;
  const float sc = dy ? 1.f : dy_scale;
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock + warp * kWarpTok;
  for (int t = 0; t < kWarpTok; ++t) {
    const int64_t k = tok0 + t;
    if (k >= n) break;
    const int ph = pos_home[k], ps = pos_send[k];
    const float pk = prob[k];
    const bf16* dsrc = dsrc_base + k * h;
    float dot = 0.f;
    for (int base = lane; base < vec; base += 32 * 4) {
      uint4 dv[4], fv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        dv[u] = make_uint4(0, 0, 0, 0);
        fv[u] = make_uint4(0, 0, 0, 0);
        if (i < vec) {
          dv[u] = ldg_stream(dsrc + i * 8);
          if (ph >= 0) fv[u] = ldg_stream(fhome + int64_t(ph) * h + i * 8);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        if (i >= vec) continue;
        float d[8], f[8];
        unpack8(dv[u], d);
        unpack8(fv[u], f);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          d[q] *= sc;
          dot = fmaf(f[q], d[q], dot);
          d[q] *= pk;
        }
        if (ps >= 0) reinterpret_cast<uint4*>(dfe + int64_t(ps) * h)[i] = pack8(d);
      }
    }
    const float dchosen = warp_sum(dot);
    const int e = expert[k];
    const float coef = dchosen * probs[k * E + e];
    for (int j = lane; j < E; j += 32)
      dlogits[k * E + j] = coef * ((j == e ? 1.f : 0.f) - probs[k * E + j]);
  }
}

// ------------------------------------------------------------------ gate backward
// replica `rep` (0 .. R.nsum-1) of token k's expert-side row, or nullptr if dropped
__device__ __forceinline__ const bf16* src_row(const RowSrc& R, int64_t k, int h, int rep = 0) {
  const int ph = R.pos_home ? R.pos_home[k] : -1;
  if (ph < 0) return nullptr;
  if (R.peers == nullptr) return R.local + int64_t(rep) * R.slot_stride + int64_t(ph) * h;
  const int e = R.expert[k];
  int c = 0;
  if (R.Tc > 1) {
    c = int(k / R.chunk_len);
    if (c >= R.Tc) c = R.Tc - 1;
  }
  const int64_t r = int64_t(ph) - R.home_base[c * R.E + e];
  const int tr = R.nsum > 1 ? rep : R.my_t;
  const bf16* base = reinterpret_cast<const bf16*>(R.peers[tr + R.Tp * (e / R.Eloc)]);
  return base + (R.pull_base[c * R.E + e] + r) * h;
}

// da[k] = dX(k) + dlogits[k] . Wg^T on the tensor cores (gate_backward's dinput,
// moe.cpp:206, plus the dispatch gradient moe.cpp:685): per warp 16 tokens x 32 columns
// per step as four mma.sync.m16n8k16 n-tiles over K = experts (16 per k-step).  dlogits
// (fp32) enter as a bf16 hi + lo pair (two MMAs, ~2^-17 relative), Wg (bf16) exactly,
// fp32 accumulation.  The n-tiles' columns are permuted so each lane ends with 8
// consecutive output columns of its two token rows: dX is read and da written as 16 B
// vectors.  Warps 0-3 / 4-7 take the two halves of the columns of a 64-token block.
// Pull variant for the peer-memory exchange (TP > 1: every dX row is the sum of T partial
// rows read over NVLink): one token row per warp-iteration, 512 B contiguous per warp load
// and four of them in flight per replica, dl . Wg^T by FMAs from smem-staged Wg.  Long
// contiguous remote reads beat the MMA variant's 64 B row segments there (0.36 vs 0.44 ms
// at C3 on 4 GPUs).
template <int EMAX>
__global__ void __launch_bounds__(kThreads) gate_bwd_dx_kernel(const RowSrc R,
                                                               const float* __restrict__ dl,
                                                               const bf16* __restrict__ wg,
                                                               int64_t n, int h, int E, int HC,
                                                               bf16* __restrict__ da) {
  extern __shared__ __align__(16) uint8_t smem[];
  bf16* s_wg = reinterpret_cast<bf16*>(smem);  // [EMAX][HC]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock + warp * kWarpTok;
  for (int c0 = 0; c0 < h; c0 += HC) {
    const int hc = min(HC, h - c0);
    __syncthreads();
    stage_wg<EMAX>(wg, E, c0, hc, HC, s_wg);
    __syncthreads();
    for (int t = 0; t < kWarpTok; ++t) {
      const int64_t k = tok0 + t;
      if (k >= n) break;
      const float d0 = lane < E ? dl[k * E + lane] : 0.f;
      const float d1 = lane + 32 < E ? dl[k * E + lane + 32] : 0.f;
      const bf16* row = src_row(R, k, h, 0);
      const bf16* src = row ? row + c0 : nullptr;
      const bf16* row1 = R.nsum > 1 && row ? src_row(R, k, h, 1) : nullptr;
      const bf16* src1 = row1 ? row1 + c0 : nullptr;
      for (int base = lane * 8; base < hc; base += 256 * 4) {
        uint4 xv[4], xv1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i0 = base + u * 256;
          xv[u] = (src && i0 < hc) ? ldg_stream(src + i0) : make_uint4(0, 0, 0, 0);
          xv1[u] = (src1 && i0 < hc) ? ldg_stream(src1 + i0) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i0 = base + u * 256;
          if (i0 >= hc) continue;
          float acc[8];
          unpack8(xv[u], acc);
          if (src1) {  // TP partial sums of the column-parallel dgrad (parallel_linear.cpp:19)
            float p1[8];
            unpack8(xv1[u], p1);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] += p1[q];
            for (int rep = 2; rep < R.nsum; ++rep) {
              unpack8(ldg_stream(src_row(R, k, h, rep) + c0 + i0), p1);
#pragma unroll
              for (int q = 0; q < 8; ++q) acc[q] += p1[q];
            }
          }
#pragma unroll
          for (int j = 0; j < EMAX; ++j) {
            const float dj = __shfl_sync(FULL, j < 32 ? d0 : d1, j & 31);
            float wv[8];
            unpack8(*reinterpret_cast<const uint4*>(s_wg + j * HC + i0), wv);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = fmaf(dj, wv[q], acc[q]);
          }
          *reinterpret_cast<uint4*>(da + k * h + c0 + i0) = pack8(acc);
        }
      }
    }
  }
}

// da = sum of the dX replicas + dl Wg^T on mma.sync.  Work unit = 128 tokens x CW hidden
// columns (CW = 512, or 256 when h % 512 != 0); persistent CTAs stride over the units, so a
// call is ~7 units per CTA slot instead of 1.7 waves of whole-row CTAs.  Per unit the CTA
// stages Wg's CW columns once in shared memory, already in the m16n8k16 B-fragment order
// (one conflict-free 8-byte LDS per lane per n-tile), and each warp streams 16 tokens x CW
// columns: dl as bf16 hi + lo A fragments (two MMAs: the product keeps ~16 mantissa bits of
// dl, fp32 accumulation), the dX rows (NS replicas) prefetched D steps of 32 columns ahead.
template <int KS, int NS, int D>
__global__ void __launch_bounds__(kThreads, 2) gate_bwd_dx_mma_kernel(const RowSrc R,
                                                                   const float* __restrict__ dl,
                                                                   const bf16* __restrict__ wg,
                                                                   int64_t n, int h, int E,
                                                                   int CW,
                                                                   bf16* __restrict__ da) {
  extern __shared__ __align__(16) uint2 s_b[];  // [CW/32 steps][4 n-tiles][KS][32 lanes]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int nchunk = h / CW, steps = CW / 32;
  const int64_t ntb = (n + 127) / 128;
  const int64_t units = ntb * nchunk;
  const int nsum = R.nsum < 1 ? 1 : R.nsum;
  int staged = -1;  // the column chunk whose fragments are in shared memory
  for (int64_t un = blockIdx.x; un < units; un += gridDim.x) {
    const int64_t tb = un / nchunk;
    const int cbeg = int(un % nchunk) * CW;
    if (cbeg != staged) {  // (with a grid that is a multiple of nchunk: once per CTA)
    __syncthreads();  // the previous unit's fragments are no longer read
    // B fragment of (step st, n-tile nt, ks) for lane (g', c'): output column
    // cbeg + 32 st + 8 (g' >> 1) + 2 nt + (g' & 1), experts 16 ks + 2 c' + {0, 1} and + 8
#pragma unroll 4
    for (int i = threadIdx.x; i < steps * 4 * KS * 32; i += kThreads) {
      const int ln = i & 31, ks = (i >> 5) % KS, nt = (i / (32 * KS)) & 3, st = i / (128 * KS);
      const int gg = ln >> 2, cc = ln & 3;
      const bf16* wrow = wg + int64_t(cbeg + 32 * st + 8 * (gg >> 1) + 2 * nt + (gg & 1)) * E;
      uint32_t b[2];
#pragma unroll
      for (int pq = 0; pq < 2; ++pq) {
        const int e0 = 16 * ks + 2 * cc + 8 * pq;
        __nv_bfloat162 wv;
        wv.x = e0 < E ? wrow[e0] : __float2bfloat16(0.f);
        wv.y = e0 + 1 < E ? wrow[e0 + 1] : __float2bfloat16(0.f);
        b[pq] = *reinterpret_cast<const uint32_t*>(&wv);
      }
      s_b[i] = make_uint2(b[0], b[1]);
    }
    __syncthreads();
    staged = cbeg;
    }
    const int64_t kr[2] = {tb * 128 + warp * 16 + g, tb * 128 + warp * 16 + g + 8};
    if (tb * 128 + warp * 16 >= n) continue;  // (every warp passed this unit's barriers)
    uint32_t ahi[KS][4], alo[KS][4];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = q & 1, pq = q >> 1;  // a0: (row g, k 2c), a1: (g+8, 2c), a2: (g, 2c+8) ...
        const int e0 = 16 * ks + 2 * c + 8 * pq;
        const int64_t k = kr[r];
        const float v0 = (k < n && e0 < E) ? dl[k * E + e0] : 0.f;
        const float v1 = (k < n && e0 + 1 < E) ? dl[k * E + e0 + 1] : 0.f;
        const __nv_bfloat162 hi = __floats2bfloat162_rn(v0, v1);
        const float2 hf = __bfloat1622float2(hi);
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
        ahi[ks][q] = *reinterpret_cast<const uint32_t*>(&hi);
        alo[ks][q] = *reinterpret_cast<const uint32_t*>(&lo);
      }
    // dX rows of this lane's two tokens, replicas 0..NS-1 -- on more than one GPU these are
    // NVLink loads from the TP replicas' buffers or the local receive slots of the push
    const bf16* rows[2][NS];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int rep = 0; rep < NS; ++rep)
        rows[r][rep] = (kr[r] < n && rep < nsum) ? src_row(R, kr[r], h, rep) : nullptr;
    const int cend = cbeg + CW;
    uint4 X[D][2][NS];
    auto load_x = [&](int col0, uint4 (&x)[2][NS]) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int rep = 0; rep < NS; ++rep)
          x[r][rep] = (rows[r][rep] && col0 < cend) ? ldg_stream(rows[r][rep] + col0 + 8 * c)
                                                    : make_uint4(0, 0, 0, 0);
    };
#pragma unroll
    for (int u = 0; u < D; ++u) load_x(cbeg + 32 * u, X[u]);
    for (int cb = cbeg; cb < cend; cb += 32 * D) {
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const int col0 = cb + 32 * u;
        const uint2* sb = s_b + ((col0 - cbeg) / 32) * (4 * KS * 32) + lane;
        float acc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const uint2 b = sb[(nt * KS + ks) * 32];
            mma_bf16_16816(acc[nt], ahi[ks][0], ahi[ks][1], ahi[ks][2], ahi[ks][3], b.x, b.y);
            mma_bf16_16816(acc[nt], alo[ks][0], alo[ks][1], alo[ks][2], alo[ks][3], b.x, b.y);
          }
        }
        // lane (g, c): row r's columns col0 + 8c .. +7 = acc[0..3][2r], acc[0..3][2r + 1]
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          if (kr[r] >= n) continue;
          float o[8], x[8];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            o[2 * nt] = acc[nt][2 * r];
            o[2 * nt + 1] = acc[nt][2 * r + 1];
          }
#pragma unroll
          for (int rep = 0; rep < NS; ++rep) {  // TP partial sums (parallel_linear.cpp:19)
            unpack8(X[u][r][rep], x);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] += x[q];
          }
          if (rows[r][0] != nullptr)
            for (int rep = NS; rep < nsum; ++rep) {  // TP > NS: the remaining replicas
              unpack8(ldg_stream(src_row(R, kr[r], h, rep) + col0 + 8 * c), x);
#pragma unroll
              for (int q = 0; q < 8; ++q) o[q] += x[q];
            }
          *reinterpret_cast<uint4*>(da + kr[r] * h + col0 + 8 * c) = pack8(o);
        }
        load_x(col0 + 32 * D, X[u]);  // refill this ring slot D steps ahead
      }
    }
  }
}


constexpr int kDwTok = 32;  // tokens per dWg partial

// dWg partials: thread owns CPT consecutive columns for all EMAX experts.
template <int EMAX, int CPT>
__global__ void __launch_bounds__(128) gate_bwd_dw_kernel(const bf16* __restrict__ a,
                                                          const float* __restrict__ dl,
                                                          int64_t n, int h, int E, int tok,
                                                          float* __restrict__ part) {
  // this CTA sums `tok` tokens (a multiple of kDwTok, staged kDwTok at a time) into one
  // partial, so the partial buffer stays small next to the activations
  __shared__ float s_dl[kDwTok * EMAX];
  const int i0 = (blockIdx.y * blockDim.x + threadIdx.x) * CPT;
  const bool col_ok = i0 < h;
  float acc[CPT][EMAX];
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int j = 0; j < EMAX; ++j) acc[c][j] = 0.f;
  for (int64_t k0 = int64_t(blockIdx.x) * tok; k0 < lmin(n, int64_t(blockIdx.x + 1) * tok);
       k0 += kDwTok) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kDwTok * EMAX; idx += blockDim.x) {
      const int t = idx / EMAX, j = idx % EMAX;
      s_dl[idx] = (k0 + t < n && j < E) ? dl[(k0 + t) * E + j] : 0.f;
    }
    __syncthreads();
    if (!col_ok) continue;
    const int tn = int(lmin(kDwTok, n - k0));
    // 8 token rows in flight per thread: loads first, then the FMAs
    for (int t0 = 0; t0 < tn; t0 += 8) {
      float xb[8][CPT];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u;
        const bf16* src = a + (k0 + t) * h + i0;
        if (t >= tn) {
#pragma unroll
          for (int c = 0; c < CPT; ++c) xb[u][c] = 0.f;
        } else if constexpr (CPT == 8) {
          float f[8];
          unpack8(ldg_stream(src), f);
#pragma unroll
          for (int c = 0; c < 8; ++c) xb[u][c] = f[c];
        } else if constexpr (CPT == 4) {
          const uint2 uu = *reinterpret_cast<const uint2*>(src);
          const float2 f0 = bf2_to_f2(uu.x), f1 = bf2_to_f2(uu.y);
          xb[u][0] = f0.x; xb[u][1] = f0.y; xb[u][2] = f1.x; xb[u][3] = f1.y;
        } else if constexpr (CPT == 2) {
          const float2 f0 = bf2_to_f2(*reinterpret_cast<const uint32_t*>(src));
          xb[u][0] = f0.x; xb[u][1] = f0.y;
        } else {
          xb[u][0] = __bfloat162float(src[0]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (t0 + u >= tn) break;
#pragma unroll
        for (int c = 0; c < CPT; ++c)
#pragma unroll
          for (int j = 0; j < EMAX; ++j)
            acc[c][j] = fmaf(xb[u][c], s_dl[(t0 + u) * EMAX + j], acc[c][j]);
      }
    }
  }
  if (!col_ok) return;
  float* out = part + (int64_t(blockIdx.x) * h + i0) * E;
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int j = 0; j < EMAX; ++j)
      if (j < E) out[c * E + j] = acc[c][j];
}

// dWg = a^T . dlogits on the tensor cores (gate_backward's dweight, moe.cpp:205):
// mma.sync.m16n8k16 with M = hidden columns, N = experts, K = tokens.  A warp owns 64
// hidden columns (four M-tiles) for a chunk of `tok` tokens; per 16-token k-step lane
// (g, c) loads 16 B (8 hidden columns at 8g) of the token rows 2c, 2c+1, 2c+8, 2c+9 and
// byte-permutes them into the A fragments: M-tile mt's rows g / g+8 are hidden columns
// 8g + 2mt / 8g + 2mt + 1 (a permutation of M undone when writing).  dlogits (fp32) enter
// as bf16 hi + lo (two MMAs, ~2^-17 relative); fp32 accumulation; one partial per chunk.
template <int NT, int D>
__global__ void __launch_bounds__(128) gate_bwd_dw_mma_kernel(const bf16* __restrict__ a,
                                                              const float* __restrict__ dl,
                                                              int64_t n, int h, int E, int tok,
                                                              float* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int hb = (blockIdx.y * 4 + warp) * 64;
  if (hb >= h) return;
  const int64_t k_beg = int64_t(blockIdx.x) * tok, k_end = lmin(n, k_beg + tok);
  float acc[4][NT][4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.f;
  const int tr[4] = {2 * c, 2 * c + 1, 2 * c + 8, 2 * c + 9};  // this lane's token rows
  // a ring of D 16-token steps in flight per warp: the token rows (64 columns = 128 B per
  // row) and the dlogits the step's B fragments are made of, both loaded D steps ahead
  // (D = 1 with 4 CTAs per SM measured fastest: 2 and 4 with fewer CTAs were 1.3-2x slower)
  uint4 X[D][4];
  float DL[D][NT][4];
  auto load = [&](int64_t k0, uint4 (&x)[4], float (&d)[NT][4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t t = k0 + tr[i];
      x[i] = t < k_end ? ldg_stream(a + t * h + hb + 8 * g) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int e = nt * 8 + g;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t t = k0 + tr[i];
        d[nt][i] = (t < k_end && e < E) ? dl[t * E + e] : 0.f;
      }
    }
  };
#pragma unroll
  for (int u = 0; u < D; ++u) load(k_beg + 16 * u, X[u], DL[u]);
  for (int64_t kb = k_beg; kb < k_end; kb += 16 * D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      // B fragments: dlogits of tokens (2c, 2c+1) and (2c+8, 2c+9) for expert nt*8 + g
      uint32_t bhi[NT][2], blo[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int pq = 0; pq < 2; ++pq) {
          const float v0 = DL[u][nt][2 * pq], v1 = DL[u][nt][2 * pq + 1];
          const __nv_bfloat162 hi = __floats2bfloat162_rn(v0, v1);
          const float2 hf = __bfloat1622float2(hi);
          const __nv_bfloat162 lo = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
          bhi[nt][pq] = *reinterpret_cast<const uint32_t*>(&hi);
          blo[nt][pq] = *reinterpret_cast<const uint32_t*>(&lo);
        }
      const uint32_t* w0 = reinterpret_cast<const uint32_t*>(&X[u][0]);
      const uint32_t* w1 = reinterpret_cast<const uint32_t*>(&X[u][1]);
      const uint32_t* w2 = reinterpret_cast<const uint32_t*>(&X[u][2]);
      const uint32_t* w3 = reinterpret_cast<const uint32_t*>(&X[u][3]);
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        // row g: hidden column 8g + 2mt (low halves), row g + 8: 8g + 2mt + 1 (high halves)
        const uint32_t a0 = __byte_perm(w0[mt], w1[mt], 0x5410);
        const uint32_t a1 = __byte_perm(w0[mt], w1[mt], 0x7632);
        const uint32_t a2 = __byte_perm(w2[mt], w3[mt], 0x5410);
        const uint32_t a3 = __byte_perm(w2[mt], w3[mt], 0x7632);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          mma_bf16_16816(acc[mt][nt], a0, a1, a2, a3, bhi[nt][0], bhi[nt][1]);
          mma_bf16_16816(acc[mt][nt], a0, a1, a2, a3, blo[nt][0], blo[nt][1]);
        }
      }
      load(kb + 16 * (u + D), X[u], DL[u]);  // refill this ring slot D steps ahead
    }
  }
  float* out = part + int64_t(blockIdx.x) * h * E;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int e = nt * 8 + 2 * c;
      const int64_t r0 = hb + 8 * g + 2 * mt, r1 = r0 + 1;
      if (e < E) {
        out[r0 * E + e] = acc[mt][nt][0];
        out[r1 * E + e] = acc[mt][nt][2];
      }
      if (e + 1 < E) {
        out[r0 * E + e + 1] = acc[mt][nt][1];
        out[r1 * E + e + 1] = acc[mt][nt][3];
      }
    }
}

// out[m] = sum_{s < ns(m)} part[s * stride + m] in a fixed order.  A CTA owns 32
// consecutive m; its 8 warps take every 8th partial with 4 independent loads in flight,
// then combine through smem.  ns(m) = ns_const, or (rows of group m / w) / rows_per_split
// when seg_off is given (column sums: partials past a group's rows are never written).
__global__ void __launch_bounds__(256) sum_partials_kernel(const float* __restrict__ part,
                                                           int64_t stride, int64_t M,
                                                           int ns_const,
                                                           const int* __restrict__ seg_off,
                                                           int w, int rows_per_split,
                                                           bf16* __restrict__ out,
                                                           int64_t out_stride) {
  __shared__ float s_acc[8][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = int64_t(blockIdx.x) * 32 + lane;
  float acc = 0.f;
  if (m < M) {
    int ns = ns_const;
    if (seg_off) {
      const int g = int(m / w);
      ns = (seg_off[g + 1] - seg_off[g] + rows_per_split - 1) / rows_per_split;
    }
    float a4[4] = {0.f, 0.f, 0.f, 0.f};
    int sidx = warp;
    for (; sidx + 24 < ns; sidx += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a4[u] += part[int64_t(sidx + 8 * u) * stride + m];
    }
    for (; sidx < ns; sidx += 8) a4[0] += part[int64_t(sidx) * stride + m];
    acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  }
  s_acc[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && m < M) {
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += s_acc[q][lane];
    out[(m / w) * out_stride + (m % w)] = __float2bfloat16(t);
  }
}

// The same reduction four columns per thread (float4 loads: 4x the bytes in flight per load
// instruction) with the identical per-column summation order as sum_partials_kernel, so
// the results are bit-identical.  Needs M, stride and w multiples of 4, part 16 B aligned.
__global__ void __launch_bounds__(256) sum_partials4_kernel(const float* __restrict__ part,
                                                            int64_t stride, int64_t M,
                                                            int ns_const,
                                                            const int* __restrict__ seg_off,
                                                            int w, int rows_per_split,
                                                            bf16* __restrict__ out,
                                                            int64_t out_stride) {
  __shared__ float4 s_acc[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = (int64_t(blockIdx.x) * 32 + lane) * 4;  // columns m .. m+3, one group
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (m < M) {
    int ns = ns_const;
    if (seg_off) {
      const int g = int(m / w);
      ns = (seg_off[g + 1] - seg_off[g] + rows_per_split - 1) / rows_per_split;
    }
    float4 a4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto add = [](float4& x, const float4 y) {
      x.x += y.x;
      x.y += y.y;
      x.z += y.z;
      x.w += y.w;
    };
    int sidx = warp;
    for (; sidx + 24 < ns; sidx += 32) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = *reinterpret_cast<const float4*>(part + int64_t(sidx + 8 * u) * stride + m);
#pragma unroll
      for (int u = 0; u < 4; ++u) add(a4[u], v[u]);
    }
    for (; sidx < ns; sidx += 8)
      add(a4[0], *reinterpret_cast<const float4*>(part + int64_t(sidx) * stride + m));
    acc.x = (a4[0].x + a4[1].x) + (a4[2].x + a4[3].x);
    acc.y = (a4[0].y + a4[1].y) + (a4[2].y + a4[3].y);
    acc.z = (a4[0].z + a4[1].z) + (a4[2].z + a4[3].z);
    acc.w = (a4[0].w + a4[1].w) + (a4[2].w + a4[3].w);
  }
  s_acc[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && m < M) {
    float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 v = s_acc[q][lane];
      t[0] += v.x;
      t[1] += v.y;
      t[2] += v.z;
      t[3] += v.w;
    }
    bf16* o = out + (m / w) * out_stride + (m % w);
#pragma unroll
    for (int c = 0; c < 4; ++c) o[c] = __float2bfloat16(t[c]);
  }
}

void sum_partials(const float* part, int64_t stride, int64_t M, int ns_const, const int* seg_off,
                  int w, int rows_per_split, bf16* out, int64_t out_stride, cudaStream_t s) {
  if (M % 4 == 0 && stride % 4 == 0 && w % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(part) & 15) == 0)
    sum_partials4_kernel<<<unsigned((M + 127) / 128), 256, 0, s>>>(part, stride, M, ns_const, seg_off, w,
                                                         rows_per_split, out, out_stride);
  else
    sum_partials_kernel<<<unsigned((M + 31) / 32), 256, 0, s>>>(part, stride, M, ns_const, seg_off, w,
                                                        rows_per_split, out, out_stride);
}

// ------------------------------------------------------------------ bias-grad column sums
constexpr int kColRows = 32;  // rows per partial

// thread = 8 columns (one 16 B vector per row), block = 128 threads = 1024 columns
__global__ void __launch_bounds__(128) colsum_part_kernel(const bf16* __restrict__ D, int64_t ld,
                                                          int w, const int* __restrict__ seg_off,
                                                          int G, int rsplits,
                                                          float* __restrict__ part) {
  const int g = blockIdx.y / rsplits, rs = blockIdx.y % rsplits;
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const int64_t r0 = int64_t(seg_off[g]) + int64_t(rs) * kColRows;
  const int64_t r1 = lmin(r0 + kColRows, seg_off[g + 1]);
  if (col >= w || r0 >= r1) return;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int64_t r = r0;
  for (; r + 8 <= r1; r += 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ldg_stream(D + (r + u) * ld + col);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float f[8];
      unpack8(v[u], f);
#pragma unroll
      for (int q = 0; q < 8; ++q) s[q] += f[q];
    }
  }
  for (; r < r1; ++r) {
    float f[8];
    unpack8(ldg_stream(D + r * ld + col), f);
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] += f[q];
  }
  float4* pp = reinterpret_cast<float4*>(part + (int64_t(rs) * G + g) * w + col);
  pp[0] = make_float4(s[0], s[1], s[2], s[3]);
  pp[1] = make_float4(s[4], s[5], s[6], s[7]);
}


// ------------------------------------------------------------------ AdamW
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ master,
                                                   float* __restrict__ m1, float* __restrict__ m2,
                                                   bf16* __restrict__ param,
                                                   const bf16* __restrict__ grad, int64_t begin,
                                                   int64_t len, float lr, float b1, float b2,
                                                   float omb1, float omb2, float eps, float wd,
                                                   float inv_c1, float inv_c2,
                                                   const float* __restrict__ coef) {
  // master/m1/m2 are indexed over the owned range; param/grad over the whole family.
  if (coef) {
    inv_c1 = coef[0];
    inv_c2 = coef[1];
  }
  const AdamK k{lr, b1, b2, omb1, omb2, eps, wd};
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += stride) {
    const float g = __bfloat162float(grad[begin + i]);
    float m = m1[i], v = m2[i], p = master[i];
    adamw_elem(p, m, v, g, k, inv_c1, inv_c2);
    m1[i] = m;
    m2[i] = v;
    master[i] = p;
    param[begin + i] = __float2bfloat16(p);
  }
}

// vectorised variant (4 elements / thread) used when everything is 16 B aligned
__global__ void __launch_bounds__(256) adam_kernel_v4(float* __restrict__ master,
                                                      float* __restrict__ m1,
                                                      float* __restrict__ m2,
                                                      bf16* __restrict__ param,
                                                      const bf16* __restrict__ grad,
                                                      int64_t begin, int64_t len4, float lr,
                                                      float b1, float b2, float omb1, float omb2,
                                                      float eps, float wd, float inv_c1,
                                                      float inv_c2, const float* __restrict__ coef) {
  if (coef) {
    inv_c1 = coef[0];
    inv_c2 = coef[1];
  }
  const AdamK k{lr, b1, b2, omb1, omb2, eps, wd};
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len4; i += stride) {
    const uint2 gu = reinterpret_cast<const uint2*>(grad + begin)[i];
    const float2 g01 = bf2_to_f2(gu.x), g23 = bf2_to_f2(gu.y);
    const float g[4] = {g01.x, g01.y, g23.x, g23.y};
    float4 mm = reinterpret_cast<float4*>(m1)[i];
    float4 vv = reinterpret_cast<float4*>(m2)[i];
    float4 pp = reinterpret_cast<float4*>(master)[i];
    float* mp = &mm.x;
    float* vp = &vv.x;
    float* pq = &pp.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      adamw_elem(pq[q], mp[q], vp[q], g[q], k, inv_c1, inv_c2);
    }
    reinterpret_cast<float4*>(m1)[i] = mm;
    reinterpret_cast<float4*>(m2)[i] = vv;
    reinterpret_cast<float4*>(master)[i] = pp;
    uint2 po;
    po.x = f2_to_bf2(pp.x, pp.y);
    po.y = f2_to_bf2(pp.z, pp.w);
    reinterpret_cast<uint2*>(param + begin)[i] = po;
  }
}

// AdamW over nseg equally sized, equally strided segments of an unsharded family
// (element e of segment k = family index k*seg_stride + seg_off + e), 4 elements per
// thread.  Used to update one tensor kind of every local expert as soon as its gradient
// is final, on a side stream, while the remaining backward GEMMs run.
__global__ void __launch_bounds__(256) adam_segments_kernel(
    float* __restrict__ master, float* __restrict__ m1, float* __restrict__ m2,
    bf16* __restrict__ param, const bf16* __restrict__ grad, int nseg, int64_t seg_stride4,
    int64_t seg_off4, int64_t seg_len4, float lr, float b1, float b2, float omb1, float omb2,
    float eps, float wd, float inv_c1, float inv_c2, const float* __restrict__ coef) {
  if (coef) {
    inv_c1 = coef[0];
    inv_c2 = coef[1];
  }
  const AdamK k{lr, b1, b2, omb1, omb2, eps, wd};
  constexpr int U = 4;  // independent 4-element vectors in flight per thread
  const int64_t total = int64_t(nseg) * seg_len4;
  // one pass of U*256 vectors per CTA (the grid covers the whole range)
  const int64_t stride = blockDim.x;
  {
    const int64_t t0 = int64_t(blockIdx.x) * blockDim.x * U + threadIdx.x;
    int64_t idx[U];
    uint2 gu[U];
    float4 mm[U], vv[U], pp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + u * stride;
      idx[u] = -1;
      if (t < total) {
        const int64_t seg = t / seg_len4;
        idx[u] = seg * seg_stride4 + seg_off4 + (t - seg * seg_len4);
        gu[u] = reinterpret_cast<const uint2*>(grad)[idx[u]];
        mm[u] = reinterpret_cast<float4*>(m1)[idx[u]];
        vv[u] = reinterpret_cast<float4*>(m2)[idx[u]];
        pp[u] = reinterpret_cast<float4*>(master)[idx[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (idx[u] < 0) continue;
      const float2 g01 = bf2_to_f2(gu[u].x), g23 = bf2_to_f2(gu[u].y);
      const float g[4] = {g01.x, g01.y, g23.x, g23.y};
      float* mp = &mm[u].x;
      float* vp = &vv[u].x;
      float* pq = &pp[u].x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        adamw_elem(pq[q], mp[q], vp[q], g[q], k, inv_c1, inv_c2);
      }
      reinterpret_cast<float4*>(m1)[idx[u]] = mm[u];
      reinterpret_cast<float4*>(m2)[idx[u]] = vv[u];
      reinterpret_cast<float4*>(master)[idx[u]] = pp[u];
      uint2 po;
      po.x = f2_to_bf2(pp[u].x, pp[u].y);
      po.y = f2_to_bf2(pp[u].z, pp[u].w);
      reinterpret_cast<uint2*>(param)[idx[u]] = po;
    }
  }
}

// AdamW over expert weight matrices whose optimizer state uses the tile-major blk_off
// layout (the unfused path of a family whose state the fused wgrad epilogue owns): one warp
// per 32x16 half block, lane = row, so both the state (contiguous 2 KB per array) and the
// row-major bf16 gradient / parameter (32 B per row) move in full sectors.
__global__ void __launch_bounds__(256) adam_tiles_kernel(
    float* __restrict__ master, float* __restrict__ m1, float* __restrict__ m2,
    bf16* __restrict__ param, const bf16* __restrict__ grad, int nseg, int64_t seg_stride,
    int64_t seg_off, int rows, int cols, float lr, float b1, float b2, float omb1, float omb2,
    float eps, float wd, float inv_c1, float inv_c2, const float* __restrict__ coef) {
  if (coef) {
    inv_c1 = coef[0];
    inv_c2 = coef[1];
  }
  const AdamK k{lr, b1, b2, omb1, omb2, eps, wd};
  const int lane = threadIdx.x & 31;
  const int64_t per_seg = int64_t(rows) * cols / 512;
  const int64_t nblk = per_seg * nseg;
  const int ntn = cols / 256;
  for (int64_t b = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; b < nblk;
       b += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t seg = b / per_seg, lb = b - seg * per_seg;
    const int64_t tile = lb >> 6;
    const int share = int(lb >> 2) & 15, hf = int(lb) & 3;
    const int64_t row = (tile / ntn) * 128 + (share >> 2) * 32 + lane;
    const int64_t col = (tile % ntn) * 256 + (share & 3) * 64 + hf * 16;
    const int64_t base = seg * seg_stride + seg_off;
    float* sm = master + base + lb * 512 + lane * 4;
    float* s1 = m1 + base + lb * 512 + lane * 4;
    float* s2 = m2 + base + lb * 512 + lane * 4;
    const int64_t pi = base + row * cols + col;
    const uint4 g0 = *reinterpret_cast<const uint4*>(grad + pi);
    const uint4 g1 = *reinterpret_cast<const uint4*>(grad + pi + 8);
    float4 w[4], a[4], c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w[j] = *reinterpret_cast<const float4*>(sm + j * 128);
      a[j] = *reinterpret_cast<const float4*>(s1 + j * 128);
      c[j] = *reinterpret_cast<const float4*>(s2 + j * 128);
    }
    const uint32_t gw[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    uint32_t pw[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 ga = bf2_to_f2(gw[2 * j]), gb = bf2_to_f2(gw[2 * j + 1]);
      const float g[4] = {ga.x, ga.y, gb.x, gb.y};
      float* pw_ = &w[j].x;
      float* pa = &a[j].x;
      float* pc = &c[j].x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        adamw_elem(pw_[q], pa[q], pc[q], g[q], k, inv_c1, inv_c2);
      }
      pw[2 * j] = f2_to_bf2(w[j].x, w[j].y);
      pw[2 * j + 1] = f2_to_bf2(w[j].z, w[j].w);
      *reinterpret_cast<float4*>(sm + j * 128) = w[j];
      *reinterpret_cast<float4*>(s1 + j * 128) = a[j];
      *reinterpret_cast<float4*>(s2 + j * 128) = c[j];
    }
    *reinterpret_cast<uint4*>(param + pi) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
    *reinterpret_cast<uint4*>(param + pi + 8) = make_uint4(pw[4], pw[5], pw[6], pw[7]);
  }
}

// steps_done += 1 and the bias corrections 1 / (1 - beta^steps_done) on the device, so a
// captured CUDA graph of the training step stays correct on every replay.
__global__ void adam_prep_kernel(long long* step, float* coef, double b1, double b2) {
  const long long st = *step + 1;
  *step = st;
  coef[0] = float(1.0 / (1.0 - pow(b1, double(st))));
  coef[1] = float(1.0 / (1.0 - pow(b2, double(st))));
}

__global__ void expert_hist_kernel(const int* __restrict__ expert, int64_t n, int E,
                                   int* __restrict__ blk_hist) {
  __shared__ int s_hist[64];
  if (threadIdx.x < 64) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t k = int64_t(blockIdx.x) * kRouteBlock + threadIdx.x;
  if (threadIdx.x < kRouteBlock && k < n) atomicAdd(&s_hist[expert[k]], 1);
  __syncthreads();
  if (threadIdx.x < E) blk_hist[int64_t(blockIdx.x) * E + threadIdx.x] = s_hist[threadIdx.x];
}

__global__ void keep_kernel(const int* __restrict__ slot, int64_t n, int64_t cap,
                            uint8_t* __restrict__ keep) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) keep[k] = slot[k] < cap ? 1 : 0;
}

__global__ void dlogits_kernel(const float* __restrict__ probs, const int* __restrict__ expert,
                               const float* __restrict__ dchosen, int64_t n, int E,
                               float* __restrict__ dl) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * E) return;
  const int64_t k = i / E;
  const int j = int(i % E), e = expert[k];
  dl[i] = dchosen[k] * probs[k * E + e] * ((j == e ? 1.f : 0.f) - probs[i]);
}

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

template <int EMAX>
int gate_hc(int h) {
  int hc = (64 * 1024) / (EMAX * 2);
  hc = hc / 256 * 256;
  return hc > h ? ((h + 255) / 256) * 256 : hc;
}

template <class K>
void smem_attr(K k, size_t bytes) {
  static std::atomic<size_t> cache[16];  // (kernel, bytes) slots; the kernel set is tiny
  static std::atomic<const void*> keys[16];
  const void* key = reinterpret_cast<const void*>(k);
  for (int i = 0; i < 16; ++i) {
    const void* cur = keys[i].load();
    if (cur == key) {
      if (cache[i].load() >= bytes) return;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
      cache[i] = bytes;
      return;
    }
    if (cur == nullptr) {
      const void* expect = nullptr;
      if (keys[i].compare_exchange_strong(expect, key) || expect == key) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
        cache[i] = bytes;
        return;
      }
    }
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

}  // namespace

// ================================================================== launchers
size_t gate_wgt_elems(int h, int E) {
  return (E >= 1 && E <= 64 && h % 64 == 0) ? size_t(gate_tc_experts(E)) * h : 0;
}

cudaError_t gate_forward(const bf16* a, const bf16* wg, int64_t n, int h, int E, float* logits,
                         float* probs, int* expert, float* prob, int* blk_hist, bf16* wgT,
                         cudaStream_t s) {
  if (E < 1 || E > 64 || h % 256 != 0) return cudaErrorInvalidValue;
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  if (wgT == nullptr || gate_wgt_elems(h, E) == 0) return cudaErrorInvalidValue;
  // tcgen05 logits (gate_sm100.cu) on the transposed gate weight
  const int em = gate_tc_experts(E);
  wg_transpose_kernel<<<ceil_div(h, 256), 256, 0, s>>>(wg, h, E, em, wgT);
  count_launch(1);
  return gate_forward_tc(a, wgT, n, h, E, logits, probs, expert, prob, blk_hist, s);
}

cudaError_t gate_route_logits(const float* logits, int64_t n, int E, float* probs, int* expert,
                              float* prob, int* blk_hist, cudaStream_t s) {
  if (E < 1 || E > 64) return cudaErrorInvalidValue;
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  route_logits_kernel<<<grid, kThreads, 0, s>>>(logits, n, E, probs, expert, prob, blk_hist);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t route_scan(const RouteScanArgs& a, cudaStream_t s) {
  if (a.E > 64 || a.T > 8 || a.T < 1) return cudaErrorInvalidValue;
  route_scan_kernel<<<1, kThreads, 0, s>>>(a);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t dispatch_rows(const bf16* a, int64_t n, int h, int E, int T, int my_chunk,
                          int64_t cap, const int* expert, const int* blk_prefix,
                          const int* chunk_prefix, const int* send_base, const int* home_base,
                          int* slot, int* pos_send, int* pos_home, bf16* xsend, cudaStream_t s) {
  if (h % 8 != 0 || E > 64) return cudaErrorInvalidValue;
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  dispatch_kernel<<<grid, kThreads, 0, s>>>(a, n, h, E, T, my_chunk, cap, expert, blk_prefix,
                                            chunk_prefix, send_base, home_base, slot, pos_send,
                                            pos_home, xsend);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t zero_pad_rows(bf16* buf, int64_t ld, int h, const int* seg_off, const int* valid,
                          int G, int max_pad_rows, cudaStream_t s) {
  if (G < 1) return cudaSuccess;
  dim3 grid(max(1, min(max_pad_rows, kPad)), G);
  zero_pad_kernel<<<grid, 128, 0, s>>>(buf, ld, h, seg_off, valid, G);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t combine_forward(const bf16* fhome, const int* pos_home, const float* prob,
                            int64_t n, int h, bf16* y, float* loss_part, cudaStream_t s) {
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  combine_fwd_kernel<<<grid, kThreads, 0, s>>>(fhome, pos_home, prob, n, h, y, loss_part);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t loss_finalize(const float* loss_part, int nblk, double inv_2n, double* loss,
                          cudaStream_t s) {
  loss_finalize_kernel<<<1, 256, 0, s>>>(loss_part, nblk, inv_2n, loss);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t combine_backward(const bf16* fhome, const int* pos_home, const int* pos_send,
                             const float* prob, const float* probs, const int* expert,
                             int64_t n, int h, int E, const bf16* dy, const bf16* y,
                             float dy_scale, bf16* dfe, float* dlogits, cudaStream_t s) {
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  combine_bwd_kernel<<<grid, kThreads, 0, s>>>(fhome, pos_home, pos_send, prob, probs, expert, n,
                                               h, E, dy, y, dy_scale, dfe, dlogits);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t gate_backward_input(const RowSrc& src, const float* dlogits, const bf16* wg,
                                int64_t n, int h, int E, bf16* da, cudaStream_t s) {
  if (E > 64 || h % 256 != 0) return cudaErrorInvalidValue;
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  // NS replicas of each dX row prefetched D steps ahead (1 = single GPU / reduced rows,
  // 2 = the TP-2 partial sums of the peer-memory exchange)
  if (src.nsum >= 2 && src.peers != nullptr) {  // NVLink pulls of TP partials: row streaming
#define TED_GBX(EM)                                                                            \
  {                                                                                            \
    const int HC = gate_hc<EM>(h);                                                             \
    const size_t sm = size_t(EM) * HC * 2;                                                     \
    smem_attr(gate_bwd_dx_kernel<EM>, sm);                                                     \
    gate_bwd_dx_kernel<EM><<<grid, kThreads, sm, s>>>(src, dlogits, wg, n, h, E, HC, da);     \
  }
    if (E <= 8) TED_GBX(8)
    else if (E <= 16) TED_GBX(16)
    else if (E <= 32) TED_GBX(32)
    else TED_GBX(64)
#undef TED_GBX
  } else {
    const int CW = h % 512 == 0 ? 512 : 256;
    const int KS = E <= 16 ? 1 : (E <= 32 ? 2 : 4);
    const size_t sm = size_t(CW / 32) * 4 * KS * 32 * sizeof(uint2);
    const int64_t units = ceil_div(n, 128) * (h / CW);
    // a grid that is a multiple of the chunk count keeps every CTA on one column chunk
    const int nch = h / CW, slots = 2 * sm_count();
    const int g2 = int(std::min<int64_t>(units, slots >= nch ? slots / nch * nch : slots));
    // local rows: one replica (1 GPU, EP-only), or the TP partials the GEMM epilogue pushed
    // into this rank's receive slots (NS = 2, a 2-step ring to stay within 128 registers)
#define TED_GDX(KSV, NSV, DV)                                                                  \
  {                                                                                            \
    smem_attr(gate_bwd_dx_mma_kernel<KSV, NSV, DV>, sm);                                      \
    gate_bwd_dx_mma_kernel<KSV, NSV, DV><<<g2, kThreads, sm, s>>>(src, dlogits, wg, n, h, E,   \
                                                                  CW, da);                     \
  }
    if (src.nsum >= 2) {
      if (KS == 1) TED_GDX(1, 2, 2)
      else if (KS == 2) TED_GDX(2, 2, 2)
      else TED_GDX(4, 2, 2)
    } else if (KS == 1) TED_GDX(1, 1, 4)
    else if (KS == 2) TED_GDX(2, 1, 4)
    else TED_GDX(4, 1, 4)
#undef TED_GDX
  }
  count_launch(1);
  return cudaGetLastError();
}

// tokens per dWg partial: enough CTAs to fill the GPU (4 per SM), as few partials as that
// allows (the partial buffer is h x E floats per token chunk)
int dw_tok(int64_t n, int h, int E) {
  // E <= 32 and h % 64 == 0: the mma.sync kernel (256 hidden columns per CTA); else FMA
  const bool mma = E <= 32 && h % 64 == 0;
  const int cpt = E <= 8 ? 8 : (E <= 16 ? 4 : (E <= 32 ? 2 : 1));
  const int64_t ycta = mma ? ceil_div(h, 256) : ceil_div(h, 128 * cpt);
  const int64_t sub = std::max<int64_t>(1, ceil_div(n, kDwTok));
  const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(sub, 4 * sm_count() / ycta));
  return int(ceil_div(sub, chunks) * kDwTok);
}

size_t gate_dw_part_floats(int64_t n, int h, int E) {
  return size_t(std::max<int64_t>(1, ceil_div(n, dw_tok(n, h, E)))) * size_t(h) * size_t(E);
}

cudaError_t gate_backward_weight(const bf16* a, const float* dlogits, int64_t n, int h, int E,
                                 float* part, bf16* dwg, cudaStream_t s) {
  if (E > 64 || h % 8 != 0) return cudaErrorInvalidValue;
  const int tok = dw_tok(n, h, E);
  const int nb = ceil_div(n, tok);
  if (nb == 0) {
    return cudaMemsetAsync(dwg, 0, sizeof(bf16) * size_t(h) * E, s);
  }
  if (E <= 32 && h % 64 == 0) {
    const dim3 grid(nb, ceil_div(h, 256));
    if (E <= 8) gate_bwd_dw_mma_kernel<1, 1><<<grid, 128, 0, s>>>(a, dlogits, n, h, E, tok, part);
    else if (E <= 16) gate_bwd_dw_mma_kernel<2, 1><<<grid, 128, 0, s>>>(a, dlogits, n, h, E, tok, part);
    else gate_bwd_dw_mma_kernel<4, 1><<<grid, 128, 0, s>>>(a, dlogits, n, h, E, tok, part);
  } else if (E <= 8) {
    gate_bwd_dw_kernel<8, 8><<<dim3(nb, ceil_div(h, 128 * 8)), 128, 0, s>>>(a, dlogits, n, h, E,
                                                                          tok, part);
  } else if (E <= 16) {
    gate_bwd_dw_kernel<16, 4><<<dim3(nb, ceil_div(h, 128 * 4)), 128, 0, s>>>(a, dlogits, n, h,
                                                                           E, tok, part);
  } else if (E <= 32) {
    gate_bwd_dw_kernel<32, 2><<<dim3(nb, ceil_div(h, 128 * 2)), 128, 0, s>>>(a, dlogits, n, h,
                                                                           E, tok, part);
  } else {
    gate_bwd_dw_kernel<64, 1><<<dim3(nb, ceil_div(h, 128)), 128, 0, s>>>(a, dlogits, n, h, E,
                                                                       tok, part);
  }
  const int64_t M = int64_t(h) * E;
  sum_partials(part, M, M, nb, nullptr, int(M), 1, dwg, 0, s);
  count_launch(2);
  return cudaGetLastError();
}

size_t colsum_part_floats(int w, int G, int max_rows_per_group) {
  return size_t(ceil_div(max_rows_per_group, kColRows)) * size_t(G) * size_t(w);
}

cudaError_t colsum_groups(const bf16* D, int64_t ld, int w, const int* seg_off, int G,
                          int max_rows_per_group, float* part, bf16* out, int64_t out_stride,
                          cudaStream_t s) {
  if (w % 8 != 0 || G < 1) return cudaErrorInvalidValue;
  const int rsplits = max(1, ceil_div(max_rows_per_group, kColRows));
  dim3 grid(ceil_div(w / 8, 128), G * rsplits);
  colsum_part_kernel<<<grid, 128, 0, s>>>(D, ld, w, seg_off, G, rsplits, part);
  const int64_t M = int64_t(G) * w;
  sum_partials(part, M, M, 0, seg_off, w, kColRows, out, out_stride, s);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t colsum_finish(const float* part, int w, const int* seg_off, int G, bf16* out,
                          int64_t out_stride, cudaStream_t s) {
  if (w % 8 != 0 || G < 1) return cudaErrorInvalidValue;
  const int64_t M = int64_t(G) * w;
  sum_partials(part, M, M, 0, seg_off, w, kColRows, out, out_stride, s);
  count_launch(1);
  return cudaGetLastError();
}

// out[k] = src[pos[k]] (zero row when pos[k] < 0): the un-permute of the dispatch gradient
// (moe.cpp:661-675) for the standalone operator; one warp per row, 16 B vectors
__global__ void __launch_bounds__(256) gather_rows_kernel(const bf16* __restrict__ src,
                                                          const int* __restrict__ pos, int64_t n,
                                                          int h, bf16* __restrict__ out) {
  const int64_t k = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (k >= n) return;
  const int lane = threadIdx.x & 31, vec = h / 8;
  const int p = pos[k];
  uint4* dst = reinterpret_cast<uint4*>(out + k * h);
  for (int i = lane; i < vec; i += 32)
    dst[i] = p >= 0 ? ldg_stream(src + int64_t(p) * h + i * 8) : make_uint4(0, 0, 0, 0);
}

cudaError_t gather_rows(const bf16* src, const int* pos, int64_t n, int h, bf16* out,
                        cudaStream_t s) {
  if (h % 8 != 0) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  gather_rows_kernel<<<ceil_div(n, 8), 256, 0, s>>>(src, pos, n, h, out);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t expert_hist(const int* expert, int64_t n, int E, int* blk_hist, cudaStream_t s) {
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  expert_hist_kernel<<<grid, kRouteBlock, 0, s>>>(expert, n, E, blk_hist);
  count_launch(1);
  return cudaGetLastError();
}

// Placement verdict of the DTD round trip (moe.cpp:537-556), computed from what the
// dispatch actually did: the reference records the kept chunk and checks that it is this
// rank's slot [t*n/T, (t+1)*n/T) -- here every token this rank dispatched (pos_send >= 0)
// must lie in chunk `slot_chunk` and every capacity-kept token of that chunk must have been
// dispatched (without DTD: slot_chunk = -1, every kept token).  verdict[0] = this
// forward's verdict, verdict[1] &= it (the rank's sticky placement_ok_, moe.cpp:553).
static __global__ void __launch_bounds__(1024) placement_verdict_kernel(
    const int* __restrict__ pos_send, const int* __restrict__ pos_home, int64_t n, int T,
    int slot_chunk, int* __restrict__ verdict) {
  const int64_t chunk = T > 1 ? n / T : n;
  int ok = 1;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    int c = T > 1 ? int(k / chunk) : 0;
    if (c >= T) c = T - 1;
    const bool expect = pos_home[k] >= 0 && (slot_chunk < 0 || c == slot_chunk);
    if ((pos_send[k] >= 0) != expect) ok = 0;
  }
  ok = __syncthreads_and(ok);
  if (threadIdx.x == 0) {
    verdict[0] = ok;
    verdict[1] &= ok;
  }
}

cudaError_t placement_verdict(const int* pos_send, const int* pos_home, int64_t n, int T,
                              int slot_chunk, int* verdict, cudaStream_t s) {
  if (n < 0 || T < 1) return cudaErrorInvalidValue;
  placement_verdict_kernel<<<1, 1024, 0, s>>>(pos_send, pos_home, n, T, slot_chunk, verdict);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t keep_from_slot(const int* slot, int64_t n, int64_t cap, uint8_t* keep,
                           cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  keep_kernel<<<ceil_div(n, 256), 256, 0, s>>>(slot, n, cap, keep);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t dlogits_from_dchosen(const float* probs, const int* expert, const float* dchosen,
                                 int64_t n, int E, float* dlogits, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  dlogits_kernel<<<ceil_div(n * E, 256), 256, 0, s>>>(probs, expert, dchosen, n, E, dlogits);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t adam_prep(long long* step, float* coef, double b1, double b2, cudaStream_t s) {
  adam_prep_kernel<<<1, 1, 0, s>>>(step, coef, b1, b2);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t adam_segments(float* master, float* m1, float* m2, bf16* param, const bf16* grad,
                          int nseg, int64_t seg_stride, int64_t seg_off, int64_t seg_len, float lr,
                          float b1, float b2, float omb1, float omb2, float eps, float wd,
                          float inv_c1, float inv_c2, const float* coef, int grid,
                          cudaStream_t s, int blk_cols) {
  if (seg_stride % 4 || seg_off % 4 || seg_len % 4 || nseg < 1) return cudaErrorInvalidValue;
  if (blk_cols > 0) {
    if (blk_cols % 256 || seg_len % (int64_t(blk_cols) * 128)) return cudaErrorInvalidValue;
    if ((seg_stride | seg_off) % 8) return cudaErrorInvalidValue;  // 16 B rows of bf16
    const int64_t blocks = int64_t(nseg) * (seg_len / 512);
    const int ctas = int(std::min<int64_t>((blocks + 7) / 8, int64_t(sm_count()) * 16));
    adam_tiles_kernel<<<ctas, 256, 0, s>>>(master, m1, m2, param, grad, nseg, seg_stride,
                                           seg_off, int(seg_len / blk_cols), blk_cols, lr, b1,
                                           b2, omb1, omb2, eps, wd, inv_c1, inv_c2, coef);
    count_launch(1);
    return cudaGetLastError();
  }
  if (seg_len == 0) return cudaSuccess;
  (void)grid;
  const int64_t items = int64_t(nseg) * (seg_len / 4);
  const int ctas = int((items + 256 * 4 - 1) / (256 * 4));
  adam_segments_kernel<<<ctas, 256, 0, s>>>(master, m1, m2, param, grad, nseg, seg_stride / 4,
                                            seg_off / 4, seg_len / 4, lr, b1, b2, omb1, omb2,
                                            eps, wd, inv_c1, inv_c2, coef);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t adam_step(float* master, float* m1, float* m2, bf16* param, const bf16* grad,
                      int64_t begin, int64_t end, int64_t tile, float lr, float b1, float b2,
                      float omb1, float omb2, float eps, float wd, float inv_c1, float inv_c2,
                      const float* coef, cudaStream_t s) {
  (void)tile;  // the tile only bounds the reference's up-cast buffer; none exists here
  const int64_t len = end - begin;
  if (len <= 0) return cudaSuccess;
  const int grid = sm_count() * 8;
  const bool v4 = (len % 4 == 0) && (begin % 4 == 0) &&
                  (reinterpret_cast<uintptr_t>(master) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(m1) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(m2) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(param) % 8 == 0) &&
                  (reinterpret_cast<uintptr_t>(grad) % 8 == 0);
  if (v4)
    adam_kernel_v4<<<grid, 256, 0, s>>>(master, m1, m2, param, grad, begin, len / 4, lr, b1, b2,
                                        omb1, omb2, eps, wd, inv_c1, inv_c2, coef);
  else
    adam_kernel<<<grid, 256, 0, s>>>(master, m1, m2, param, grad, begin, len, lr, b1, b2, omb1,
                                     omb2, eps, wd, inv_c1, inv_c2, coef);
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace ted
