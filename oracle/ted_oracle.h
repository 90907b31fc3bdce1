/* ted_oracle.h -- TEST INFRASTRUCTURE ONLY: a CPU restatement (fp64, plain C) of the
 * reference's MoE-layer hot path, used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the CHECKER.  The product never links this.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libtedsim_ref.so, built from /root/reference by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 * Capacity-factor overflow has no reference counterpart and is
 * "parity unpinned" -- see DESIGN.md section 3.
 */
#ifndef TED_ORACLE_H
#define TED_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

uint64_t o_mix_seed(uint64_t seed, const char* tag);                     /* tensor.cpp:100-111 */
void o_seeded_init(double* out, int64_t n, uint64_t seed, double scale); /* tensor.cpp:113-129 */
void o_gate_route_logits(const double* logits, int64_t n, int E, int* expert, double* chosen,
                         double* probs); /* moe.cpp:166-184 */
void o_gate_forward(const double* a, const double* wg, int64_t n, int h, int E, double* logits,
                    int* expert, double* chosen, double* probs); /* moe.cpp:158-186 */
void o_gate_backward(const double* a, const double* wg, const double* probs, const int* expert,
                     const double* dchosen, int64_t n, int h, int E, double* dwg,
                     double* dinput); /* moe.cpp:188-208 */
int64_t o_capacity(double cf, int64_t n, int E);
void o_route_capacity(const int* expert, int64_t n, int E, int64_t cap, int T, int* slot,
                      uint8_t* keep, int* kept_counts /* [T][E] */);
double o_gelu(double x);      /* nn.cpp:92-97  */
double o_gelu_grad(double x); /* nn.cpp:99-106 */
/* MoE branch fwd+bwd over S source shards of n tokens each (all experts local, like
 * SerialModel::forward_layer/backward_layer, moe.cpp:973-1075), extended with the
 * per-shard capacity drop.  dy == NULL -> dy = y / N (loss sum(y^2)/(2N), moe.cpp:379-391). */
int o_moe_layer(int S, int64_t n, int h, int f, int E, double cf, const double* a,
                const double* wg, const double* w1, const double* b1, const double* w2,
                const double* b2, const double* dy_in, double* y, double* loss, double* da,
                double* dwg, double* dw1, double* db1, double* dw2, double* db2, int* expert,
                int* slot, uint8_t* keep, double* logits, double* probs);
void o_shard_range(int64_t total, int parts, int index, int64_t* begin, int64_t* end);
/* OptimizerShard::step_owned (optimizer.cpp:58-104): one step over the owned range.
 * Returns the up-cast peak bytes the reference accounts (4 * min(tile, owned)). */
uint64_t o_adam_step_owned(int64_t begin, int64_t end, int64_t step, double lr, double b1,
                           double b2, double eps, double wd, int tiles_enabled,
                           int64_t tile_size, const double* grad_full, double* master,
                           double* m1, double* m2, double* out_full);
#ifdef __cplusplus
}
#endif
#endif
