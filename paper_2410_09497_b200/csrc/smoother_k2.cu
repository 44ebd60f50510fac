// K3 instantiation for degree 2 (see smoother_kernel.cuh).
#include "smoother_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_SMOOTH(2)
}  // namespace smg
