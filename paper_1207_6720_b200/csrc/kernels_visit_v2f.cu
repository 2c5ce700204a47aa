// One lane type of the fused visit kernel (V2<float> lanes over float fields).
#include "visit_impl.cuh"

namespace fmgsr {
template void visit_fill_launch<V2<float>, float, SHAPE_WIDE>(const VisitDesc<float>&, cudaStream_t);
}  // namespace fmgsr
