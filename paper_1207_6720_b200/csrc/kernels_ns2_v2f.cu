// One lane type of the V(2,2) smoother kernel (V2<float> lanes over float fields).
#include "ns2_impl.cuh"

namespace fmgsr {
template void ns2_fill_launch<V2<float>, float>(const Ns2Desc<float>&, cudaStream_t);
}  // namespace fmgsr
