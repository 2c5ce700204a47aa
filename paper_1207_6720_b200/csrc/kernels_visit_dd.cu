// One lane type of the fused visit kernel (double lanes over double fields), deep-ring shape.
#include "visit_impl.cuh"

namespace fmgsr {
template void visit_fill_launch<double, double, SHAPE_DEEP>(const VisitDesc<double>&, cudaStream_t);
}  // namespace fmgsr
