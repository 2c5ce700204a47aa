// One lane type of the V(2,2) smoother kernel (double lanes over double fields).
#include "ns2_impl.cuh"

namespace fmgsr {
template void ns2_fill_launch<double, double>(const Ns2Desc<double>&, cudaStream_t);
}  // namespace fmgsr
