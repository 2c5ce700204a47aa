// fp32 fields, fp64 arithmetic: double lanes over float storage (both shapes).
#include "visit_impl.cuh"

namespace fmgsr {
template void visit_fill_launch<double, float, SHAPE_WIDE, float>(const VisitDesc<float>&, cudaStream_t);
template void visit_fill_launch<double, float, SHAPE_DEEP, float>(const VisitDesc<float>&, cudaStream_t);
}  // namespace fmgsr
