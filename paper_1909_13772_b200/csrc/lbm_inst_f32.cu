// fp32 storage of (f - w_i), fp64 register arithmetic (FMA contraction allowed:
// this variant is compared against the fp64 oracle with a relative
// tolerance, not bitwise).
#define LBM_REAL float
#define LBM_UNIT unit_f32
#include "lbm_inst.cuh"

namespace lbm {
LBM_DEFINE_MRT_SETTER(set_mrt_tables_f32)
}
