// fp64 storage, fp64 arithmetic.  Build with -fmad=false: every operation is
// rounded on its own, matching the numpy reference kernel bit for bit.
#define LBM_REAL double
#define LBM_UNIT unit_f64
#include "lbm_inst.cuh"

namespace lbm {
LBM_DEFINE_MRT_SETTER(set_mrt_tables_f64)
}
