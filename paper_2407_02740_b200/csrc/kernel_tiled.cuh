// kernel_tiled.cuh -- layout TILED_REG (placeholder until the register-tiled kernel lands).
#pragma once
#include "common.cuh"

static inline bool tiled_supported(int, int, int, int, int) { return false; }

template <class PartialsFn>
static int launch_tiled(cudaStream_t, int, size_t, EvalParams &, int *, const char **, PartialsFn) { return -4; }
