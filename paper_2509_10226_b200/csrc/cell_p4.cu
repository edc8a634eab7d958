// Cell-kernel instantiations, degree 4.
#include "cell_launch.cuh"

namespace tmf {
TMF_CELL_TU(35, 70)
}  // namespace tmf
