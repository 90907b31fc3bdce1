// peer_kernels.cu -- the EP all-to-all, the DTD all-gathers and the combine's return trip
// done by the routing kernels themselves over NVLink peer memory (CUDA IPC mappings of
// the expert ranks' assembled buffers), instead of staging + NCCL send/recv.
//
//   dispatch (moe.cpp:454-493):  every kept row of this rank's DTD chunk is stored
//       straight into its expert's assembled buffer on replica my_t -- or, with DTD, on
//       every TP replica (the all-gather folded into the scatter: one source per row).
//   return + combine (moe.cpp:504-563): each token pulls its expert's output row from
//       every TP replica and sums the partials in fp32 -- the row-parallel all-reduce
//       (parallel_linear.cpp:28) folded into the consumer -- then scales by p; the row is
//       also kept in a token-ordered local copy for the backward (dchosen = <f_home, dy>).
//   backward dispatch (moe.cpp:603-632): p * dy rows stored into the experts' dFe buffers
//       exactly like the forward dispatch; the return of dX (with the column-parallel
//       dgrad's TP partial sums, parallel_linear.cpp:19) is a pull in gate backward.
// Ordering across ranks: plane barriers through IPC-mapped flag arrays (below; NCCL
// all-reduce barriers with TED_BARRIER=nccl); every writer kernel ends with a system-scope
// fence.  plan_peer builds the exchange plan on the device.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ted_internal.h"
#include "ted_plan.h"
#include "ted_vec.cuh"

namespace ted {
namespace {

constexpr int kThreads = 256;
constexpr int kWarpTok = kRouteBlock / 8;


// Row r of this token on replica t of expert e's EP rank.
__device__ __forceinline__ bf16* dst_row(const PeerDst& D, int t, int e, int64_t r, int h) {
  bf16* base = reinterpret_cast<bf16*>(D.peers[t + D.Tp * (e / D.Eloc)]);
  return base + (D.disp_base[e] + r) * h;
}

__device__ __forceinline__ void scale8(uint4& u, float s) {
  float f[8];
  unpack8(u, f);
#pragma unroll
  for (int q = 0; q < 8; ++q) f[q] *= s;
  u = pack8(f);
}

__global__ void __launch_bounds__(kThreads) scatter_peer_kernel(const bf16* __restrict__ a,
                                                                const int* __restrict__ pos_send,
                                                                const int* __restrict__ expert,
                                                                int64_t n, int h, PeerDst D,
                                                                const float* __restrict__ scale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = h / 8;
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock + warp * kWarpTok;
  for (int t = 0; t < kWarpTok; ++t) {
    const int64_t k = tok0 + t;
    if (k >= n) break;
    const int ps = pos_send[k];
    if (ps < 0) continue;
    const int e = expert[k];
    const int64_t r = int64_t(ps) - D.send_base[e];
    if (D.clamp_rows && r >= D.clamp_rows[e]) continue;
    const float sc = scale ? scale[k] : 1.f;
    const uint4* src = reinterpret_cast<const uint4*>(a + k * h);
    const int t0 = D.all_replicas ? 0 : D.my_t;
    const int t1 = D.all_replicas ? D.Tp : D.my_t + 1;
    for (int base = lane; base < vec; base += 32 * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        if (i < vec) {
          v[u] = ldg_stream(src + i);
          if (scale) scale8(v[u], sc);
        }
      }
      for (int tr = t0; tr < t1; ++tr) {
        if ((D.part == 1 && tr != D.my_t) || (D.part == 2 && tr == D.my_t)) continue;
        uint4* dst = reinterpret_cast<uint4*>(dst_row(D, tr, e, r, h));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = base + u * 32;
          if (i < vec) dst[i] = v[u];
        }
      }
    }
  }
  __threadfence_system();
}

__device__ __forceinline__ const bf16* pull_row(const RowSrc& R, int64_t k, int h, int rep) {
  const int ph = R.pos_home[k];
  if (ph < 0) return nullptr;
  if (R.peers == nullptr)  // pushed partials in this rank's receive slots
    return R.local + int64_t(rep) * R.slot_stride + int64_t(ph) * h;
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

__global__ void __launch_bounds__(kThreads) combine_pull_kernel(RowSrc R,
                                                                const float* __restrict__ prob,
                                                                int64_t n, int h,
                                                                bf16* __restrict__ y,
                                                                bf16* __restrict__ fhome,
                                                                float* __restrict__ loss_part) {
  __shared__ float s_red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = h / 8;
  float sq = 0.f;
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock + warp * kWarpTok;
  for (int t = 0; t < kWarpTok; ++t) {
    const int64_t k = tok0 + t;
    if (k >= n) break;
    const bf16* src = pull_row(R, k, h, 0);
    // row-parallel GEMM2: sum the TP partial rows here instead of an all-reduce
    const bf16* src1 = (R.nsum > 1 && src) ? pull_row(R, k, h, 1) : nullptr;
    const float pk = prob[k];
    uint4* yd = reinterpret_cast<uint4*>(y + k * h);
    uint4* fd = reinterpret_cast<uint4*>(fhome + k * h);
    for (int base = lane; base < vec; base += 32 * 4) {
      uint4 v[4], v1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        v[u] = make_uint4(0, 0, 0, 0);
        v1[u] = make_uint4(0, 0, 0, 0);
        if (i < vec && src) v[u] = ldg_stream(reinterpret_cast<const uint4*>(src) + i);
        if (i < vec && src1) v1[u] = ldg_stream(reinterpret_cast<const uint4*>(src1) + i);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        if (i >= vec) continue;
        float f[8];
        unpack8(v[u], f);
        if (src1) {
          float g[8];
          unpack8(v1[u], g);
#pragma unroll
          for (int q = 0; q < 8; ++q) f[q] += g[q];
          for (int rep = 2; rep < R.nsum; ++rep) {
            unpack8(ldg_stream(reinterpret_cast<const uint4*>(pull_row(R, k, h, rep)) + i), g);
#pragma unroll
            for (int q = 0; q < 8; ++q) f[q] += g[q];
          }
          v[u] = pack8(f);
        }
        fd[i] = v[u];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          f[q] *= pk;
          sq = fmaf(f[q], f[q], sq);
        }
        yd[i] = pack8(f);
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

__global__ void __launch_bounds__(kThreads) combine_bwd_peer_kernel(
    const bf16* __restrict__ fhome, const int* __restrict__ pos_home,
    const int* __restrict__ pos_send, const float* __restrict__ prob,
    const float* __restrict__ probs, const int* __restrict__ expert, int64_t n, int h, int E,
    const bf16* __restrict__ dy, const bf16* __restrict__ y, float dy_scale, PeerDst D,
    float* __restrict__ dlogits) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = h / 8;
  const bf16* dsrc_base = dy ? dy : y;
  const float sc = dy ? 1.f : dy_scale;
  const int64_t tok0 = int64_t(blockIdx.x) * kRouteBlock + warp * kWarpTok;
  for (int t = 0; t < kWarpTok; ++t) {
    const int64_t k = tok0 + t;
    if (k >= n) break;
    const int ph = pos_home[k], ps = pos_send[k];
    const int e = expert[k];
    const float pk = prob[k];
    const uint4* dsrc = reinterpret_cast<const uint4*>(dsrc_base + k * h);
    const uint4* fsrc = reinterpret_cast<const uint4*>(fhome + k * h);
    const int64_t r = ps >= 0 ? int64_t(ps) - D.send_base[e] : 0;
    const bool send = ps >= 0 && !(D.clamp_rows && r >= D.clamp_rows[e]);
    const int t0 = D.all_replicas ? 0 : D.my_t;
    const int t1 = !send ? t0 : (D.all_replicas ? D.Tp : D.my_t + 1);
    float dot = 0.f;
    for (int base = lane; base < vec; base += 32 * 4) {
      uint4 dv[4], fv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32;
        dv[u] = make_uint4(0, 0, 0, 0);
        fv[u] = make_uint4(0, 0, 0, 0);
        if (i < vec) {
          dv[u] = ldg_stream(dsrc + i);
          if (ph >= 0) fv[u] = ldg_stream(fsrc + i);
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
        dv[u] = pack8(d);
      }
      for (int tr = t0; tr < t1; ++tr) {
        uint4* dst = reinterpret_cast<uint4*>(dst_row(D, tr, e, r, h));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = base + u * 32;
          if (i < vec) dst[i] = dv[u];
        }
      }
    }
    const float dchosen = warp_sum(dot);
    const float coef = dchosen * probs[k * E + e];
    for (int j = lane; j < E; j += 32)
      dlogits[k * E + j] = coef * ((j == e ? 1.f : 0.f) - probs[k * E + j]);
  }
  __threadfence_system();
}

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

}  // namespace

cudaError_t scatter_rows_peer(const bf16* a, const int* pos_send, const int* expert, int64_t n,
                              int h, const PeerDst& dst, const float* scale, bool scale_by_prob,
                              cudaStream_t s) {
  if (h % 8 != 0) return cudaErrorInvalidValue;
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  scatter_peer_kernel<<<grid, kThreads, 0, s>>>(a, pos_send, expert, n, h, dst,
                                                scale_by_prob ? scale : nullptr);
  count_launch(1);
  return cudaGetLastError();
}

// Plane barrier over NVLink peer memory: thread i publishes `epoch` into slot `me` of
// member i's flag array (system-scope release after a system fence, so every earlier
// peer store of this GPU is visible first), then waits until member i's epoch has
// arrived in this GPU's own array (system-scope acquire).  A member that does not arrive
// within timeout_ns (the reference's collective_timeout, moe.hpp:96; 0 = wait forever,
// measured on the global nanosecond timer, independent of the SM clock) is recorded in
// *fault (1 + its plane rank; host-mapped, read by the host as TimeoutError) and the
// kernel returns instead of trapping, so the CUDA context survives.  Once a fault is
// recorded every later barrier returns at once (the step's data are void; the host
// reports the error at its next call).
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void plane_barrier_kernel(const unsigned long long* __restrict__ flags, int PS,
                                     int me, unsigned* __restrict__ epoch_dev,
                                     int* __restrict__ fault, unsigned long long timeout_ns) {
  // the epoch lives on the device (every member runs the same barrier sequence), so a
  // captured CUDA graph of the step advances it on every replay
  __shared__ unsigned s_epoch;
  __shared__ int s_fault;
  const int i = threadIdx.x;
  if (i == 0) {
    s_epoch = *epoch_dev + 1;
    *epoch_dev = s_epoch;
    s_fault = *reinterpret_cast<volatile int*>(fault);
  }
  __threadfence_system();
  __syncthreads();
  if (s_fault) return;
  const unsigned epoch = s_epoch;
  if (i < PS) {
    unsigned* dst = reinterpret_cast<unsigned*>(flags[i]) + me;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
    const unsigned* mine = reinterpret_cast<const unsigned*>(flags[me]) + i;
    const unsigned long long t0 = global_ns();
    unsigned v = 0;
    for (unsigned spin = 0;; ++spin) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (int(v - epoch) >= 0) break;
      if ((spin & 255) == 255) {
        if (timeout_ns != 0 && global_ns() - t0 > timeout_ns) {
          atomicCAS(fault, 0, 1 + i);  // member i never arrived: a peer is gone or stalled
          __threadfence_system();
          break;
        }
        if (*reinterpret_cast<volatile int*>(fault)) break;  // another slot timed out
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

cudaError_t plane_barrier_peer(const unsigned long long* flags, int PS, int me,
                               unsigned* epoch_dev, int* fault, unsigned long long timeout_ns,
                               cudaStream_t s) {
  if (PS < 1 || PS > 1024 || fault == nullptr) return cudaErrorInvalidValue;
  plane_barrier_kernel<<<1, ((PS + 31) / 32) * 32, 0, s>>>(flags, PS, me, epoch_dev, fault,
                                                          timeout_ns);
  count_launch(1);
  return cudaGetLastError();
}

// The peer-exchange plan on the device (ted_plan.h's offsets, no host round trip): from the
// plane-gathered chunk counts (member t + T*ep contributes [Tc][E]; TP peers route
// identical tokens, so the t = 0 members' counts are the sources' counts) compute this
// rank's assembled segments (seg_off[Eloc+1], then valid rows [Eloc]) and, for every
// expert e, where this rank's rows land in e's assembled buffer: disp_base[e] (my chunk)
// and pull_base[c][e] (every chunk c, for the return pulls).  One thread per expert.
__global__ void plan_peer_kernel(const int* __restrict__ kc_all, int T, int P, int E, int Tc,
                                 int my_ep, int my_c, int* __restrict__ seg,
                                 long long* __restrict__ disp_base,
                                 long long* __restrict__ pull_base) {
  const int e = threadIdx.x;
  if (e < E) peer_plan_expert(kc_all, T, P, E, Tc, my_ep, my_c, e, disp_base, pull_base, seg);
}

cudaError_t plan_peer(const int* kc_all, int T, int P, int E, int Tc, int my_ep, int my_c,
                      int* seg, long long* disp_base, long long* pull_base, cudaStream_t s) {
  if (E < 1 || E > 1024 || E % P != 0) return cudaErrorInvalidValue;
  plan_peer_kernel<<<1, ((E + 31) / 32) * 32, 0, s>>>(kc_all, T, P, E, Tc, my_ep, my_c, seg,
                                                     disp_base, pull_base);
  count_launch(1);
  return cudaGetLastError();
}

// The reference's CommLedger entries of one MoE pass on this rank (fabric.cpp:163-287
// accounting, per member: calls + 1 and this member's payload per collective; summing the
// members gives the reference's group records).  The exchange itself may be fused into
// NVLink kernels; the ledger records the collectives the reference runs for the same data
// (moe.cpp:435-563 / :582-686): dispatch and return all-to-all over EP (P > 1), the DTD
// expert-side and home all-gathers over TP, the expert block's TP all-reduce (T > 1).
// led: [phase][op][calls, bytes], op order AllReduce, AllGather, AllToAll (types.hpp:39).
__global__ void ledger_moe_pass_kernel(unsigned long long* __restrict__ led, int phase, int P,
                                       int T, int dtd, int Tc, int E, int Eloc, int my_t,
                                       int my_ep, const int* __restrict__ kc,
                                       const int* __restrict__ kc_all, int src_stride,
                                       const int* __restrict__ seg_valid, int h) {
  if (threadIdx.x != 0) return;
  long long valid = 0, send = 0, recv = 0;
  for (int le = 0; le < Eloc; ++le) valid += seg_valid[le];
  const int my_c = dtd ? my_t : 0;
  for (int e = 0; e < E; ++e) send += kc[my_c * E + e];
  if (dtd) {  // my block of the expert-side rows: chunk my_t of every EP source
    for (int s = 0; s < P; ++s)
      for (int le = 0; le < Eloc; ++le)
        recv += kc_all[(size_t(src_stride) * s * Tc + my_t) * E + my_ep * Eloc + le];
  } else {
    recv = valid;
  }
  const unsigned long long hb = 2ull * h;
  unsigned long long* row = led + size_t(phase) * 3 * 2;
  if (T > 1) {  // AllReduce (expert block, row-parallel partial sums)
    row[0] += 1;
    row[1] += (unsigned long long)valid * hb;
  }
  if (dtd) {  // AllGather: the expert-side block and the home chunk
    row[2] += 2;
    row[3] += (unsigned long long)(recv + send) * hb;
  }
  if (P > 1) {  // AllToAll: dispatch (my rows, self segments included) and return
    row[4] += 2;
    row[5] += (unsigned long long)(send + recv) * hb;
  }
}

cudaError_t ledger_moe_pass(unsigned long long* led, int phase, int P, int T, int dtd, int Tc,
                            int E, int Eloc, int my_t, int my_ep, const int* kc, const int* kc_all,
                            int src_stride, const int* seg_valid, int h, cudaStream_t s) {
  ledger_moe_pass_kernel<<<1, 32, 0, s>>>(led, phase, P, T, dtd, Tc, E, Eloc, my_t, my_ep, kc,
                                          kc_all, src_stride, seg_valid, h);
  count_launch(1);
  return cudaGetLastError();
}

// Where every row of this rank's assembled buffer goes back to (the push return of the
// GEMM2 / dgrad1 epilogues): local expert le's segment holds blocks (chunk c, source s)
// of C(s, c, e) rows in that order (peer_plan_expert); their home rows on every TP member
// of source shard s are home_base_s(c, e) + i, home_base_s(c, e) = rows of source s's
// chunks before c + rows of chunk c for experts before e (route_scan's home layout).
// row_home = -1 for the segment's pad rows.  One CTA per local expert.
__global__ void push_map_kernel(const int* __restrict__ kc_all, int T, int P, int E, int Tc,
                                int my_ep, const int* __restrict__ seg, int* __restrict__ row_home,
                                int* __restrict__ row_src) {
  const int Eloc = E / P, le = blockIdx.x, e = my_ep * Eloc + le;
  auto C = [&](int s_, int c, int ee) { return kc_all[(int64_t(T) * s_ * Tc + c) * E + ee]; };
  __shared__ int s_start[64 * 8], s_cnt[64 * 8], s_home[64 * 8];
  const int nb = Tc * P;  // <= 8 * 64
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int c = b / P, s_ = b % P;
    int hb = 0;
    for (int c2 = 0; c2 < c; ++c2)
      for (int e2 = 0; e2 < E; ++e2) hb += C(s_, c2, e2);
    for (int e2 = 0; e2 < e; ++e2) hb += C(s_, c, e2);
    s_home[b] = hb;
    s_cnt[b] = C(s_, c, e);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int r = seg[le];
    for (int b = 0; b < nb; ++b) {
      s_start[b] = r;
      r += s_cnt[b];
    }
  }
  __syncthreads();
  for (int b = 0; b < nb; ++b) {
    const int st = s_start[b], cnt = s_cnt[b], hb = s_home[b], s_ = b % P;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      row_home[st + i] = hb + i;
      row_src[st + i] = s_;
    }
  }
  const int end = seg[le] + seg[Eloc + 1 + le];
  const int seg_end = le + 1 < Eloc ? seg[le + 1] : seg[Eloc];
  for (int r = end + threadIdx.x; r < seg_end; r += blockDim.x) row_home[r] = -1;
}

cudaError_t push_map(const int* kc_all, int T, int P, int E, int Tc, int my_ep, const int* seg,
                     int* row_home, int* row_src, cudaStream_t s) {
  if (E % P != 0 || Tc * P > 64 * 8) return cudaErrorInvalidValue;
  push_map_kernel<<<E / P, 256, 0, s>>>(kc_all, T, P, E, Tc, my_ep, seg, row_home, row_src);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t combine_pull(const RowSrc& src, const float* prob, int64_t n, int h, bf16* y,
                         bf16* fhome, float* loss_part, cudaStream_t s) {
  if (h % 8 != 0 || (src.peers == nullptr && src.local == nullptr)) return cudaErrorInvalidValue;
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  combine_pull_kernel<<<grid, kThreads, 0, s>>>(src, prob, n, h, y, fhome, loss_part);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t combine_backward_peer(const bf16* fhome, const int* pos_home, const int* pos_send,
                                  const float* prob, const float* probs, const int* expert,
                                  int64_t n, int h, int E, const bf16* dy, const bf16* y,
                                  float dy_scale, const PeerDst& dst, float* dlogits,
                                  cudaStream_t s) {
  if (h % 8 != 0) return cudaErrorInvalidValue;
  const int grid = ceil_div(n, kRouteBlock);
  if (grid == 0) return cudaSuccess;
  combine_bwd_peer_kernel<<<grid, kThreads, 0, s>>>(fhome, pos_home, pos_send, prob, probs,
                                                    expert, n, h, E, dy, y, dy_scale, dst,
                                                    dlogits);
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace ted
