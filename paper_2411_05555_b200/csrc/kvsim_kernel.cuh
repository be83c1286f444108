// kvsim_kernel.cuh — kernel K3 (the persistent warp-per-point sweep), shared
// by the lean (kvsim_sweep.cu) and full (kvsim_sweep_full.cu) translation units.
#pragma once
#include "kvsim_sim.cuh"

// MINB = minimum resident blocks per SM requested from ptxas (register cap
// 65536 / (128 * MINB)); selected at context open (KVSIM_MINB, default below).
// FULL = false: the lean sweep kernel (plain points only); true: every
// specialisation (events, detail metrics, AcceLLM extensions, SPEC variants).
template <int MINB, bool FULL>
__global__ void __launch_bounds__(kvsim_dev::kWarpsPerBlock * 32, MINB) kvsim_sweep_kernel(const __grid_constant__ kvsim_dev::SweepArgs a) {
  kvsim_dev::WarpScratch* scratch = reinterpret_cast<kvsim_dev::WarpScratch*>(kvsim_smem);
  const int w = threadIdx.x >> 5;
  const int64_t slot = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
#if defined(KVSIM_SIM_SMEM)
  // block-shared copy of the parameters (kvsim_sim.cuh: AR)
  if (threadIdx.x == 0) kvsim_dev::kvsim_args_smem = a;
  __syncthreads();
  if (slot >= a.slots) return;
  kvsim_dev::sweep_warp<FULL>(&kvsim_dev::kvsim_args_smem, &scratch[w], (int32_t)slot);
#else
  if (slot >= a.slots) return;
  kvsim_dev::sweep_warp<FULL>(&a, &scratch[w], (int32_t)slot);
#endif
}

