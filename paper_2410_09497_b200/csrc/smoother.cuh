// Per-degree entry points of the patch smoother kernel (one translation unit per degree so the
// heavily unrolled instantiations compile in parallel).
#pragma once
#include "smg_internal.cuh"

namespace smg {
template <int K>
void smooth_launch_k(Context& ctx, int level, int prec, int colour, void* x, const void* r, int zlo, int zhi, int vz0,
                     int vz1);
template <int K>
void smooth_fused_launch_k(Context& ctx, int level, int prec, int colour, void* x_out, const void* x_in,
                           const void* b);
}  // namespace smg
