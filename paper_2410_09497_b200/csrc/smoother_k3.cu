// K3 instantiation for degree 3 (see smoother_kernel.cuh).
#include "smoother_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_SMOOTH(3)
}  // namespace smg
