// Cell-kernel instantiations, degree 1.
#include "cell_launch.cuh"

namespace tmf {
TMF_CELL_TU(4, 4)
TMF_CELL_TU(4, 5)
TMF_CELL_TU(4, 1)   // modal tables (M = 1)
}  // namespace tmf
