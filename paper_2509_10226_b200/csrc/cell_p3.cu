// Cell-kernel instantiations, degree 3.
#include "cell_launch.cuh"

namespace tmf {
TMF_CELL_TU(20, 35)
}  // namespace tmf
