// Per-kernel clocks / power / time at the C3 wgrad shape (tools/, not part of the product).
// Each phase loops one kernel for ~`secs` seconds while tools/wgrad_power.sh samples
// nvidia-smi; the phase boundaries are printed as wall-clock milliseconds so the samples
// can be attributed.  Links the product library for the kernels themselves.
//   phases: fwd   = GEMM1 forward (ROWS, bias+GELU)              -- tensor-bound control
//           wgrad = wgrad1 with the plain store epilogue (bf16 dW1)
//           fused = wgrad1 with the fused AdamW epilogue (the step's dominant kernel)
//           adam  = the unfused AdamW over the same parameters (tile-major state)
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2303_06318_b200/csrc
//        tools/wgrad_power.cu -o tools/wgrad_power -L paper_2303_06318_b200 -lted_b200
//        -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2303_06318_b200'
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ted_internal.h"

using namespace ted;

static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::system_clock::now().time_since_epoch())
      .count();
}

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

__global__ void fill_k(bf16* p, int64_t n, float s, uint32_t seed) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x = uint32_t(i) * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = __float2bfloat16(s * ((x & 0xffff) / 32768.f - 1.f));
  }
}

int main(int argc, char** argv) {
  const int h = argc > 1 ? atoi(argv[1]) : 4096;
  const int f = argc > 2 ? atoi(argv[2]) : 16384;
  const int G = argc > 3 ? atoi(argv[3]) : 16;
  const double secs = argc > 4 ? atof(argv[4]) : 3.0;
  const char* only = argc > 5 ? argv[5] : "";
  std::vector<int> off(G + 1, 0);
  for (int g = 0; g < G; ++g) off[g + 1] = off[g] + ((g & 1) ? 2176 : 2048);
  const int rows = off[G];
  int* d_off;
  CK(cudaMalloc(&d_off, (G + 1) * sizeof(int)));
  CK(cudaMemcpy(d_off, off.data(), (G + 1) * sizeof(int), cudaMemcpyHostToDevice));
  const int64_t P = int64_t(G) * h * f;
  bf16 *X, *H, *Z, *W1, *b1, *prm, *grd;
  float *mst, *m1, *m2, *coef;
  CK(cudaMalloc(&X, size_t(rows) * h * 2));
  CK(cudaMalloc(&H, size_t(rows) * f * 2));
  CK(cudaMalloc(&Z, size_t(rows) * f * 2));
  CK(cudaMalloc(&W1, size_t(P) * 2));
  CK(cudaMalloc(&b1, size_t(G) * f * 2));
  CK(cudaMalloc(&prm, size_t(P) * 2));
  CK(cudaMalloc(&grd, size_t(P) * 2));
  CK(cudaMalloc(&mst, size_t(P) * 4));
  CK(cudaMalloc(&m1, size_t(P) * 4));
  CK(cudaMalloc(&m2, size_t(P) * 4));
  CK(cudaMalloc(&coef, 8));
  fill_k<<<1184, 256>>>(X, int64_t(rows) * h, 1.f, 1);
  fill_k<<<1184, 256>>>(H, int64_t(rows) * f, 1.f, 2);
  fill_k<<<1184, 256>>>(W1, P, 0.02f, 3);
  fill_k<<<1184, 256>>>(b1, int64_t(G) * f, 0.1f, 4);
  CK(cudaMemset(mst, 0, size_t(P) * 4));
  CK(cudaMemset(m1, 0, size_t(P) * 4));
  CK(cudaMemset(m2, 0, size_t(P) * 4));
  const float c[2] = {10.f, 1000.f};
  CK(cudaMemcpy(coef, c, 8, cudaMemcpyHostToDevice));
  CK(cudaDeviceSynchronize());
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  AdamK ak{1e-4f, 0.9f, 0.999f, 0.1f, 0.001f, 1e-8f, 0.01f};

  auto launch = [&](const char* ph) -> cudaError_t {
    const char* why = nullptr;
    if (!strcmp(ph, "fwd")) {
      GemmOperands o{X, h, false, W1, f, int64_t(h) * f, true};
      GemmParams p{};
      p.mode = GEMM_ROWS;
      p.epi = EPI_BIAS_GELU;
      p.groups = G;
      p.M = 0;
      p.N = f;
      p.K = h;
      p.seg_off = d_off;
      p.C = Z;
      p.ldc = f;
      p.bias = b1;
      p.bias_group_stride = f;
      p.aux = H;
      p.ld_aux = f;
      cudaError_t e = grouped_gemm(o, p, rows, s, &why);
      if (why) fprintf(stderr, "%s\n", why);
      return e;
    }
    if (!strcmp(ph, "adam"))
      return adam_segments(mst, m1, m2, prm, grd, G, int64_t(h) * f, 0, int64_t(h) * f, ak.lr,
                           ak.b1, ak.b2, ak.omb1, ak.omb2, ak.eps, ak.wd, 10.f, 1000.f, coef,
                           sm_count() * 4, s, f);
    const bool fused = !strcmp(ph, "fused");
    GemmOperands o{X, h, true, H, f, 0, true};
    GemmParams p{};
    p.mode = GEMM_KDIM;
    p.epi = fused ? EPI_ADAM : EPI_STORE;
    p.groups = G;
    p.M = h;
    p.N = f;
    p.K = 0;
    p.seg_off = d_off;
    p.C = fused ? prm : grd;
    p.ldc = f;
    p.c_group_stride = int64_t(h) * f;
    if (fused) {
      p.adam_master = mst;
      p.adam_m1 = m1;
      p.adam_m2 = m2;
      p.adam_coef = coef;
      p.adam = ak;
    }
    cudaError_t e = grouped_gemm(o, p, rows, s, &why);
    if (why) fprintf(stderr, "%s\n", why);
    return e;
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char* phases[] = {"fwd", "wgrad", "fused", "adam"};
  for (const char* ph : phases) {
    if (only[0] && !strstr(only, ph)) continue;
    for (int i = 0; i < 3; ++i) CK(launch(ph));
    CK(cudaStreamSynchronize(s));
    // calibrate launches per phase
    CK(cudaEventRecord(e0, s));
    CK(launch(ph));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms1 = 0;
    CK(cudaEventElapsedTime(&ms1, e0, e1));
    const int iters = std::max(3, int(secs * 1000 / ms1));
    const double t0 = now_ms();
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < iters; ++i) CK(launch(ph));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    const double t1 = now_ms();
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double per = ms / iters;
    double flops = 0, bytes = 0;
    if (!strcmp(ph, "fwd")) flops = 2.0 * rows * h * double(f), bytes = rows * (2.0 * h + 4.0 * f);
    else if (!strcmp(ph, "wgrad")) flops = 2.0 * rows * h * double(f), bytes = 2.0 * rows * (h + f) + 2.0 * P;
    else if (!strcmp(ph, "fused")) flops = 2.0 * rows * h * double(f), bytes = 2.0 * rows * (h + f) + 26.0 * P;
    else bytes = 26.0 * P;
    printf("PHASE %s start_ms %.0f end_ms %.0f iters %d ms_per_launch %.4f TFLOPs %.1f GBps %.1f\n",
           ph, t0, t1, iters, per, flops / per / 1e9, bytes / per / 1e6);
    fflush(stdout);
  }
  return 0;
}
