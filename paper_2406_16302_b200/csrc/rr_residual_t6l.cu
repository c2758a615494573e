// rr_residual_t6l.cu -- the residual kernels of rr_residual.cu instantiated once more with T6's direction
// sampled "uniformly toward the light" (technique (6); RR_T6_TOWARD_LIGHT render flag; SURVEY 8(f)
// row 4).  Every path's ghost crossings then carry the direction density p_dir(d | x_G) of the path's direction
// through them (the queries know which way the path runs an edge), so T6's candidate pdf follows; a separate
// translation unit keeps every branch of the variant out of the default kernels (namespace rr::kt6l).
#define RR_T6L_KERNELS 1
#include "rr_residual.cu"
