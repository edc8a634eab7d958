// Cell-kernel instantiations, degree 2.
#include "cell_launch.cuh"

namespace tmf {
TMF_CELL_TU(10, 14)
TMF_CELL_TU(10, 15)
TMF_CELL_TU(10, 4)   // modal tables (M = dim P_{p-1} unit-weight points)
}  // namespace tmf
