// Match kernels (lanes, converge, ceiling) of table layout 6 (global_u16); see kernels.cu.
#define DFA_TU_MODE 6
#include "kernels.cu"
