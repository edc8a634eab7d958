// Cell-kernel instantiations, degree 3.
#include "cell_launch.cuh"

namespace tmf {
TMF_CELL_TU(20, 35)
TMF_CELL_TU(20, 10)   // modal tables (M = dim P_{p-1} unit-weight points)
}  // namespace tmf
