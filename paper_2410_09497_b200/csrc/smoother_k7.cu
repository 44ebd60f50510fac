// K3 instantiation for degree 7 (see smoother_kernel.cuh).
#include "smoother_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_SMOOTH(7)
}  // namespace smg
