// One lane type of the fused visit kernel (V2<double> lanes over double
// fields) in the R4 launch shape (4-pair ring, four CTAs per SM).
#include "visit_impl.cuh"

namespace fmgsr {
template void visit_fill_launch<V2<double>, double, SHAPE_R4>(const VisitDesc<double>&, cudaStream_t);
}  // namespace fmgsr
