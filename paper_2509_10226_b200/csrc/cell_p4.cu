// Cell-kernel instantiations, degree 4.
#include "cell_launch.cuh"

namespace tmf {
TMF_CELL_TU(35, 70)
TMF_CELL_TU(35, 20)   // modal tables (M = dim P_{p-1} unit-weight points)
}  // namespace tmf
