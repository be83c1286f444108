// kvsim_sweep_full.cu — the full sweep kernel K3<3, FULL = true>: every
// specialisation (event logs, detail metrics, AcceLLM timer extensions, the
// optional SPEC variants). Its handlers stay outlined
// (KVSIM_OUTLINE_HANDLERS): inlining them into eight specialisations would
// multiply its compile time, and these runs (parity checks, reports) are
// not the sweep hot path. The lean kernel (kvsim_sweep.cu) inlines them.
#ifndef KVSIM_LEAN_ONLY
#define KVSIM_OUTLINE_HANDLERS 1
#include "kvsim_kernel.cuh"

template __global__ void kvsim_sweep_kernel<3, true>(const __grid_constant__ kvsim_dev::SweepArgs);

using SweepFn = void (*)(kvsim_dev::SweepArgs);
SweepFn kvsim_full_kernel(int /*minb*/) { return kvsim_sweep_kernel<3, true>; }
#endif
