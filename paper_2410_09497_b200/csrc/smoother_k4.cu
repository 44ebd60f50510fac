// K3 instantiation for degree 4 (see smoother_kernel.cuh).
#include "smoother_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_SMOOTH(4)
}  // namespace smg
