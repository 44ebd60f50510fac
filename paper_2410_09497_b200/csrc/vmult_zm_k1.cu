// K1z (z-march operator, vmult_zm.cuh) instantiation for degree 1.
#include "vmult_zm.cuh"

namespace smg {
SMG_INSTANTIATE_ZM(1)
}  // namespace smg
