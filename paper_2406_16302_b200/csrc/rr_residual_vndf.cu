// rr_residual_vndf.cu -- the residual kernels of rr_residual.cu instantiated once more with GGX
// visible-normal sampling compiled in (RR_VNDF render flag; Heitz 2018).  A separate
// translation unit keeps every branch of the variant out of the default kernels (namespace rr::kvndf).
#define RR_VNDF_KERNELS 1
#include "rr_residual.cu"
