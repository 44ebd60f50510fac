// K1z (z-march operator, vmult_zm.cuh) instantiation for degree 2.
#include "vmult_zm.cuh"

namespace smg {
SMG_INSTANTIATE_ZM(2)
}  // namespace smg
