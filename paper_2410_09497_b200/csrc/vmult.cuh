// Per-degree entry points of the Stokes vmult kernel (one translation unit per degree so the heavy
// template instantiations compile in parallel).
#pragma once
#include "smg_internal.cuh"

namespace smg {
template <int K>
void vmult_launch_k(Context& ctx, int level, int prec, const VmultArgs& a);
template <int K>
void vmult_upload_k(const double* t, const float* f);
// z-march kernel (vmult_zm.cuh, k <= 2): returns false when it does not handle the launch
template <int K>
bool zm_vmult_launch_k(Context& ctx, int level, int prec, const VmultArgs& a);
template <int K>
void zm_upload_k(const double* t, const float* f);
}  // namespace smg
