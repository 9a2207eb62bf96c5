// veq_eval.cu — K2 evaluator translation unit: k_eval_warp and its launcher
// (see veq_kernels.cuh). Split from veq_api.cu so the two compile in
// parallel.
#define VEQ_TU_EVAL
#include "veq_kernels.cuh"

namespace veqd {

void eval_warp_config(int smem, int *per_sm) {
  cudaFuncSetAttribute(k_eval_warp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_eval_warp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  *per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_eval_warp<false>, EVAL_BLOCK, smem);
  int p2 = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, k_eval_warp<true>, EVAL_BLOCK, smem);
  if (p2 < *per_sm) *per_sm = p2;
}

void launch_eval_warp(uint32_t grid, uint32_t block, int smem, cudaStream_t s, const Batch &B, const Table &T,
                      const EvalCtx &E, const uint4 *desc, const unsigned long long *n_work_dev,
                      unsigned long long *cursor, char *pool, unsigned long long *pool_used, uint64_t pool_cap,
                      uint64_t chunk, bool defer) {
  if (defer)
    k_eval_warp<true><<<grid, block, smem, s>>>(B, T, E, desc, n_work_dev, cursor, pool, pool_used, pool_cap, chunk);
  else
    k_eval_warp<false><<<grid, block, smem, s>>>(B, T, E, desc, n_work_dev, cursor, pool, pool_used, pool_cap, chunk);
}

}  // namespace veqd
