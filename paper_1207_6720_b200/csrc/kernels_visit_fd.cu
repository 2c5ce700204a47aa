// One lane type of the fused visit kernel (float lanes over float fields), deep-ring shape.
#include "visit_impl.cuh"

namespace fmgsr {
template void visit_fill_launch<float, float, SHAPE_DEEP>(const VisitDesc<float>&, cudaStream_t);
}  // namespace fmgsr
