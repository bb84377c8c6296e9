/*
 * ttkv_dropin_c.h -- C entry points of libttkv.so (the C++ drop-in) for FFI
 * consumers that need the reference's deterministic input generator.
 *
 *   ttkv_generate_workload   generate_workload (workload.cpp:42-95):
 *                            Gaussian or planted-needle stream, mt19937_64
 *                            Box-Muller, bit-identical to the reference.
 */
#ifndef TTKV_DROPIN_C_H
#define TTKV_DROPIN_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Arrays are caller-owned: pre_k[ctx][d_k], pre_v[ctx][d_v], dec_k[T][d_k],
 * dec_v[T][d_v], dec_q[T][d_k].  Returns TTKV_OK or TTKV_ECONFIG. */
int ttkv_generate_workload(int needle, uint64_t ctx, uint64_t T, uint32_t d_k, uint32_t d_v,
                           uint64_t seed, uint64_t needle_block_position, double needle_strength,
                           float* pre_k, float* pre_v, float* dec_k, float* dec_v, float* dec_q);

#ifdef __cplusplus
}
#endif
#endif
