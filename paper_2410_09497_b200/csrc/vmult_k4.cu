// K1/K2 instantiation for degree 4 (see vmult_kernel.cuh).
#include "vmult_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_VMULT(4)
}  // namespace smg
