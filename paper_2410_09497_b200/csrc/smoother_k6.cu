// K3 instantiation for degree 6 (see smoother_kernel.cuh).
#include "smoother_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_SMOOTH(6)
}  // namespace smg
