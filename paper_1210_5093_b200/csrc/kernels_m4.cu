// Match kernels (lanes, converge, ceiling) of table layout 4 (window_u16); see kernels.cu.
#define DFA_TU_MODE 4
#include "kernels.cu"
