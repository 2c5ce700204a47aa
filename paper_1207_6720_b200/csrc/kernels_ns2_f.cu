// One lane type of the V(2,2) smoother kernel (float lanes over float fields).
#include "ns2_impl.cuh"

namespace fmgsr {
template void ns2_fill_launch<float, float>(const Ns2Desc<float>&, cudaStream_t);
}  // namespace fmgsr
