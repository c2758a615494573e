// rr_residual_var.cu -- the residual kernels of rr_residual.cu instantiated once more with the mapping / sampling
// variants of SURVEY 8(f) row 4 compiled in, each selected at run time by its render flag:
//  * RR_T6_TOWARD_LIGHT (technique (6)): T6's direction "uniformly toward the light"; every path's
//    ghost crossings then carry the direction density p_dir(d | x_G) of the path's direction through them (the
//    queries know which way the path runs an edge), so T6's candidate pdf follows;
//  * RR_TOBJ_MIDPATH ("transform with object movement"): the first mid-path hit of a moved object
//    maps to the same object-space point in the other state instead of being replayed.
// A separate translation unit keeps every branch of the variants out of the default kernels (namespace
// rr::kvar), whose code generation is unchanged.
#define RR_VAR_KERNELS 1
#include "rr_residual.cu"
