// K1/K2 instantiation for degree 1 (see vmult_kernel.cuh).
#include "vmult_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_VMULT(1)
}  // namespace smg
