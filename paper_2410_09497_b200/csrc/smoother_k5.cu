// K3 instantiation for degree 5 (see smoother_kernel.cuh).
#include "smoother_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_SMOOTH(5)
}  // namespace smg
