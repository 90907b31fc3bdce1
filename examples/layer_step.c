/* examples/layer_step.c -- the reference-side integration in plain C: one rank's TED MoE
 * layer created from the reference's config structs, trained for a few steps through the
 * C ABI (include/ted.h).  Device buffers come from the CUDA runtime; the layer never sees
 * a torch type.
 *
 *   gcc -std=c11 -I include examples/layer_step.c -L paper_2303_06318_b200 -lted_b200 \
 *       -L/usr/local/cuda/lib64 -lcudart -o layer_step
 */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "ted.h"

#define CHECK(x)                                                        \
  do {                                                                  \
    int rc_ = (x);                                                      \
    if (rc_ != TED_OK) {                                                \
      fprintf(stderr, "%s -> %d: %s\n", #x, rc_, ted_last_error());     \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main(void) {
  ted_model_cfg model;
  ted_topo_cfg topo;
  ted_flags flags;
  ted_adam_cfg adam;
  ted_tile_cfg tiles;
  ted_default_configs(&model, &topo, &flags, &adam, &tiles);
  model.hidden = 1024;
  model.experts = 8;
  model.tokens_per_shard = 4096;
  ted_layer* layer = NULL;
  CHECK(ted_layer_create(&model, &topo, &flags, &adam, &tiles, 1.25, 1, 0, NULL, &layer));
  CHECK(ted_layer_init_params(layer, 1234));
  const size_t elems = (size_t)model.tokens_per_shard * (size_t)model.hidden;
  uint16_t *a = NULL, *y = NULL, *da = NULL;
  if (cudaMalloc((void**)&a, elems * 2) != cudaSuccess || cudaMalloc((void**)&y, elems * 2) ||
      cudaMalloc((void**)&da, elems * 2))
    return 1;
  cudaMemset(a, 0x3c, elems * 2); /* bf16 ~1.0 tokens */
  for (int step = 0; step < 3; ++step) {
    double loss = 0.0;
    CHECK(ted_layer_step(layer, a, y, da, NULL));
    CHECK(ted_layer_loss(layer, &loss, NULL));
    printf("step %d loss %.6f\n", step, loss);
  }
  ted_layer_destroy(layer);
  cudaFree(a);
  cudaFree(y);
  cudaFree(da);
  return 0;
}
