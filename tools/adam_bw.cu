// Bandwidth ceiling of the AdamW access mix on this GPU (tools/, not part of the product):
// copy (1 read + 1 write stream) vs the AdamW pattern (fp32 master/m/v read+write, bf16
// grad read, bf16 param write = 26 B/element), each with U independent vectors per thread.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/adam_bw.cu -o tools/adam_bw
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

template <int U>
__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, int64_t n4) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * U;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x * U + threadIdx.x; i < n4; i += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * blockDim.x < n4) v[u] = a[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * blockDim.x < n4) b[i + u * blockDim.x] = v[u];
  }
}

template <int U>
__global__ void adam_k(float4* __restrict__ w, float4* __restrict__ m, float4* __restrict__ v,
                       const uint2* __restrict__ g, uint2* __restrict__ p, int64_t n4) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * U;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x * U + threadIdx.x; i < n4; i += stride) {
    float4 a[U], b[U], c[U];
    uint2 gg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = i + u * blockDim.x;
      if (k < n4) {
        a[u] = w[k];
        b[u] = m[k];
        c[u] = v[k];
        gg[u] = g[k];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = i + u * blockDim.x;
      if (k >= n4) continue;
      const float gr = __uint_as_float(gg[u].x << 16);
      float* pa = &a[u].x;
      float* pb = &b[u].x;
      float* pc = &c[u].x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pb[q] = 0.9f * pb[q] + 0.1f * gr;
        pc[q] = 0.999f * pc[q] + 0.001f * gr * gr;
        pa[q] -= 1e-4f * (pb[q] / (sqrtf(pc[q]) + 1e-8f) + 0.01f * pa[q]);
      }
      w[k] = a[u];
      m[k] = b[u];
      v[k] = c[u];
      __nv_bfloat162 lo = __floats2bfloat162_rn(a[u].x, a[u].y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(a[u].z, a[u].w);
      p[k] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
}

// The fused wgrad epilogue's state traffic alone: one CTA per SM, NW warps, each warp
// walks its 32-row x 128-column share of the CTA's 128x256 tiles as eight 32x16 half blocks
// (blk_off layout: 2 KB per array, lane = row), DEPTH halves of state in registers.
__device__ __forceinline__ int64_t blk_off(int64_t r, int64_t c, int64_t cols) {
  return ((r >> 5) * (cols >> 4) + (c >> 4)) * 512 + ((c >> 2) & 3) * 128 + (r & 31) * 4 +
         (c & 3);
}
template <int NW, int DEPTH, int LAYOUT>
__global__ void __launch_bounds__(NW * 32, 1)
    epi_sim(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
            int groups, int M, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = N / 256, per = (M / 128) * nt, total = groups * per;
  const int WPT = NW / 8;  // warps sharing one 32x128 share (split the 8 halves)
  const int sp = (warp / WPT) & 3, chalf = (warp / WPT) >> 2, sub = warp % WPT;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int g = t / per, l = t % per, mb = l / nt, nb = l % nt;
    const int row0 = mb * 128 + sp * 32, colw = nb * 256 + chalf * 128;
    const int64_t base = int64_t(g) * M * N + lane * 4;
    // LAYOUT 1: tile-major -- tile t's 64 half blocks contiguous (warp share 16 KB)
    const int64_t tbase = int64_t(t) * (128 * 256) + int64_t((sp + 4 * chalf) * 8) * 512 +
                          lane * 4;
#define OFF(hh) (LAYOUT == 0 ? base + blk_off(row0, colw + 16 * (hh), N) \
                             : tbase + int64_t(hh) * 512)
    float4 st[DEPTH][12];
    const int nh = 8 / WPT;
#pragma unroll
    for (int d = 0; d < DEPTH - 1; ++d) {
      const int64_t o = OFF(sub * nh + d);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        st[d][j] = *reinterpret_cast<const float4*>(w + o + j * 128);
        st[d][4 + j] = *reinterpret_cast<const float4*>(m + o + j * 128);
        st[d][8 + j] = *reinterpret_cast<const float4*>(v + o + j * 128);
      }
    }
#pragma unroll
    for (int k = 0; k < nh; ++k) {
      if (k + DEPTH - 1 < nh) {
        const int kk = k + DEPTH - 1;
        const int64_t o = OFF(sub * nh + kk);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          st[kk % DEPTH][j] = *reinterpret_cast<const float4*>(w + o + j * 128);
          st[kk % DEPTH][4 + j] = *reinterpret_cast<const float4*>(m + o + j * 128);
          st[kk % DEPTH][8 + j] = *reinterpret_cast<const float4*>(v + o + j * 128);
        }
      }
      float4(&c)[12] = st[k % DEPTH];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float* a = &c[j].x;
        float* b = &c[4 + j].x;
        float* q = &c[8 + j].x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          b[e] = 0.9f * b[e] + 0.1f * a[e];
          q[e] = 0.999f * q[e] + 0.001f * a[e] * a[e];
          a[e] -= 1e-4f * (b[e] / (sqrtf(q[e]) + 1e-8f));
        }
      }
      const int64_t o = OFF(sub * nh + k);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        *reinterpret_cast<float4*>(w + o + j * 128) = c[j];
        *reinterpret_cast<float4*>(m + o + j * 128) = c[4 + j];
        *reinterpret_cast<float4*>(v + o + j * 128) = c[8 + j];
      }
    }
  }
}

// Epilogue walk with quarter half tiles (32 rows x 8 columns: 24 state registers) and NW
// warps per CTA sharing the four TMEM sub-partitions unevenly (NW/4 warps per sub-partition
// split the 256 columns into NW/4 runs of 8-column quarters)
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    epi_sim_q(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
              int groups, int M, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int WPS = NW / 4;       // warps per sub-partition
  constexpr int NQ = 256 / 8;       // quarters per tile row block
  const int sp = warp % 4, k = warp / 4;
  const int q0 = (NQ * k) / WPS, q1 = (NQ * (k + 1)) / WPS;
  const int nt = N / 256, per = (M / 128) * nt, total = groups * per;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int64_t tbase = int64_t(t) * (128 * 256) + lane * 4;
    for (int q = q0; q < q1; ++q) {
      // tile-major: quarter q of sub-partition sp = half (q / 2) of the warp share, chunk pair
      const int cc = q * 8;  // column in the tile
      const int share = sp * 4 + (cc >> 6), half = (cc >> 4) & 3, jc = (cc >> 2) & 3;
      const int64_t o = tbase + (int64_t(share) * 4 + half) * 512 + jc * 128;
      float4 a0 = *reinterpret_cast<const float4*>(w + o), a1 = *reinterpret_cast<const float4*>(w + o + 128);
      float4 b0 = *reinterpret_cast<const float4*>(m + o), b1 = *reinterpret_cast<const float4*>(m + o + 128);
      float4 c0 = *reinterpret_cast<const float4*>(v + o), c1 = *reinterpret_cast<const float4*>(v + o + 128);
      float* A[2] = {&a0.x, &a1.x};
      float* B[2] = {&b0.x, &b1.x};
      float* Cc[2] = {&c0.x, &c1.x};
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          B[u][e] = 0.9f * B[u][e] + 0.1f * A[u][e];
          Cc[u][e] = 0.999f * Cc[u][e] + 0.001f * A[u][e] * A[u][e];
          A[u][e] -= 1e-4f * (B[u][e] / (sqrtf(Cc[u][e]) + 1e-8f));
        }
      *reinterpret_cast<float4*>(w + o) = a0;
      *reinterpret_cast<float4*>(w + o + 128) = a1;
      *reinterpret_cast<float4*>(m + o) = b0;
      *reinterpret_cast<float4*>(m + o + 128) = b1;
      *reinterpret_cast<float4*>(v + o) = c0;
      *reinterpret_cast<float4*>(v + o + 128) = c1;
    }
  }
}

int main() {
  const int64_t n = int64_t(64) << 20;  // elements (fp32 arrays of 256 MB)
  const int64_t n4 = n / 4;
  float4 *w, *m, *v, *a, *b;
  uint2 *g, *p;
  cudaMalloc(&w, n * 4);
  cudaMalloc(&m, n * 4);
  cudaMalloc(&v, n * 4);
  cudaMalloc(&g, n * 2);
  cudaMalloc(&p, n * 2);
  cudaMalloc(&a, n * 16);
  cudaMalloc(&b, n * 16);
  cudaMemset(w, 0, n * 4);
  cudaMemset(m, 0, n * 4);
  cudaMemset(v, 0, n * 4);
  cudaMemset(g, 0, n * 2);
  cudaMemset(a, 0, n * 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    const int it = 20;
    for (int i = 0; i < it; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.3f ms  %7.1f GB/s\n", name, ms / it, bytes / (ms / it * 1e-3) / 1e9);
  };
  const double cb = double(n) * 16 * 2;
  for (int mult : {4, 8, 16}) {
    const int grid = sms * mult;
    char nm[64];
    snprintf(nm, 64, "copy U4 grid=%dxSM", mult);
    run(nm, cb, [&] { copy_k<4><<<grid, 256>>>(a, b, n4 * 4); });
  }
  const double ab = double(n) * 26;
  for (int mult : {2, 4, 8, 16}) {
    const int grid = sms * mult;
    char nm[64];
    snprintf(nm, 64, "adam U1 grid=%dxSM", mult);
    run(nm, ab, [&] { adam_k<1><<<grid, 256>>>(w, m, v, g, p, n4); });
    snprintf(nm, 64, "adam U2 grid=%dxSM", mult);
    run(nm, ab, [&] { adam_k<2><<<grid, 256>>>(w, m, v, g, p, n4); });
    snprintf(nm, 64, "adam U4 grid=%dxSM", mult);
    run(nm, ab, [&] { adam_k<4><<<grid, 256>>>(w, m, v, g, p, n4); });
  }
  {  // C2 wgrad1 shape: 8 groups of 1024 x 4096 (24 B/element of fp32 state traffic)
    const int G = 8, M = 1024, N = 4096;
    const double eb = double(G) * M * N * 24;
    float* W = reinterpret_cast<float*>(w);
    float* Mm = reinterpret_cast<float*>(m);
    float* V = reinterpret_cast<float*>(v);
#define EPI(NW, D, LY)                                                                    \
  run("epi_sim " #NW " warps depth " #D " layout " #LY, eb,                                \
      [&] { epi_sim<NW, D, LY><<<sms, NW * 32>>>(W, Mm, V, G, M, N); });
    EPI(8, 1, 0) EPI(8, 2, 0) EPI(16, 1, 0) EPI(16, 2, 0)
    EPI(8, 1, 1) EPI(8, 2, 1) EPI(16, 1, 1) EPI(16, 2, 1) EPI(32, 1, 1)
#define EPQ(NW) run("epi_sim_q " #NW " warps (quarters, uneven)", eb, \
      [&] { epi_sim_q<NW><<<sms, NW * 32>>>(W, Mm, V, G, M, N); });
    EPQ(16) EPQ(20) EPQ(24) EPQ(28) EPQ(32)
    const int64_t n1 = int64_t(G) * M * N;
    run("flat adam (same size) U1 8xSM", n1 * 26.0,
        [&] { adam_k<1><<<sms * 8, 256>>>(w, m, v, g, p, n1 / 4); });
  }
  const cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
