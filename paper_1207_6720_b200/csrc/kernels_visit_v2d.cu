// One lane type of the fused visit kernel (V2<double> lanes over double fields).
#include "visit_impl.cuh"

namespace fmgsr {
template void visit_fill_launch<V2<double>, double, SHAPE_WIDE>(const VisitDesc<double>&, cudaStream_t);
}  // namespace fmgsr
