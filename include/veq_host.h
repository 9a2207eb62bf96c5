/* veq_host.h — C-ABI of the host-side frontend (libveq_host.so).
 *
 * Replaces the reference's kernel-IR loader
 *   ctaeq::parse_kernel / parse_config / elaborate
 *   (proj/include/ctaeq/frontend.hpp:104-129, called at pipeline.cpp:150-169)
 * and make_symbolic_inputs (pipeline.hpp:73-74): it turns kernel sources and
 * a launch configuration into packed IR batches (VEQIR02 byte images, see
 * include/veq_ir.hpp) ready for veq_load_batch. Elaboration is per CTA;
 * a grid is elaborated block-parallel on host threads.
 */
#ifndef VEQ_HOST_H
#define VEQ_HOST_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { VEQH_OK = 0, VEQH_E_KERNEL_A = 1, VEQH_E_KERNEL_B = 2, VEQH_E_CONFIG = 3, VEQH_E_ARG = 4,
       VEQH_E_TEMPLATE = 5 /* grid not expressible as one template (caller elaborates per CTA) */ };

/* One result: two VEQIR02 images (kernel A, kernel B) and the input symbol
 * table as text lines "name<TAB>size". Free with veqh_free. */
typedef struct veqh_pair {
  uint8_t *ir_a;
  size_t ir_a_len;
  uint8_t *ir_b;
  size_t ir_b_len;
  char *inputs;
} veqh_pair;

/* Elaborates kernel_a / kernel_b under cfg for n_blocks CTAs: block k binds
 * params.<block_param> = block_base + k (block_param NULL: the config as
 * given). Batch program k is block k. On error returns VEQH_E_* and writes a
 * message in the reference's wording to err. */
int veqh_elaborate_grid(const char *kernel_a, const char *kernel_b, const char *cfg, const char *block_param,
                        uint32_t block_base, uint32_t n_blocks, uint32_t n_workers, int want_names, veqh_pair *out,
                        char *err, size_t errlen);

void veqh_free(veqh_pair *p);

/* A grid as ONE template program per kernel plus per-CTA array shifts.
 * Elaborating with params.<block_param> symbolic (it may flow into array
 * offsets only, possibly through quotients/remainders by constants) yields a
 * block-independent program; CTA b (b < n_blocks, block value block_base + b)
 * is that program with every Load/Store offset on array a shifted by
 * deltas[b * n_arrays + a] — byte-identical to its own elaboration by
 * veqh_elaborate_grid. The device expands the template per CTA
 * (veq_instantiate), so a grid's IR crosses PCIe once. Returns
 * VEQH_E_TEMPLATE (err: why) when control, constants or sync sets depend on
 * the block, or an array shifts non-uniformly. Free with veqh_free_template. */
typedef struct veqh_template {
  uint8_t *ir_a;
  size_t ir_a_len;
  uint8_t *ir_b;
  size_t ir_b_len;
  char *inputs;
  int32_t *deltas_a; /* [n_blocks * n_arrays_a] */
  int32_t *deltas_b; /* [n_blocks * n_arrays_b] */
  uint32_t n_arrays_a, n_arrays_b, n_blocks;
} veqh_template;

int veqh_elaborate_template(const char *kernel_a, const char *kernel_b, const char *cfg, const char *block_param,
                            int64_t block_base, uint32_t n_blocks, int want_names, veqh_template *out, char *err,
                            size_t errlen);
void veqh_free_template(veqh_template *p);

/* ctaeq::parse_config (proj/include/ctaeq/frontend.hpp:120,
 * proj/src/frontend.cpp:1017-1110): on success writes the parsed launch
 * configuration as "key=value" lines (threads, threads_a, threads_b,
 * warp_size, params.<name> in name order, inputs, outputs) and returns
 * VEQH_OK; on error returns VEQH_E_CONFIG with the reference's ParseError
 * text ("<line>:1: <message>"). */
int veqh_parse_config(const char *cfg, char *out, size_t outlen);

#ifdef __cplusplus
}
#endif
#endif
