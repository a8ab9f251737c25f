// Match kernels (lanes, converge, ceiling) of table layout 3 (window_u8); see kernels.cu.
#define DFA_TU_MODE 3
#include "kernels.cu"
