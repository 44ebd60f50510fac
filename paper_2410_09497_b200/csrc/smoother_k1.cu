// K3 instantiation for degree 1 (see smoother_kernel.cuh).
#include "smoother_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_SMOOTH(1)
}  // namespace smg
