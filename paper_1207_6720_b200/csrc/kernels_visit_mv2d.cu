// fp32 fields, fp64 arithmetic: V2<double> lanes over V2<float> storage.
#include "visit_impl.cuh"

namespace fmgsr {
template void visit_fill_launch<V2<double>, float, SHAPE_WIDE, V2<float>>(const VisitDesc<float>&,
                                                                           cudaStream_t);
}  // namespace fmgsr
