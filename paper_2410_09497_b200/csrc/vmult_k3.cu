// K1/K2 instantiation for degree 3 (see vmult_kernel.cuh).
#include "vmult_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_VMULT(3)
}  // namespace smg
