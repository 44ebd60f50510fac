// K1/K2 instantiation for degree 4 (see vmult_kernel.cuh).
#define SMG_TUNE 1  // round-1 tuning: alternative brick shapes via SMG_VMULT_VARIANT
#include "vmult_kernel.cuh"

namespace smg {
SMG_INSTANTIATE_VMULT(4)
}  // namespace smg
