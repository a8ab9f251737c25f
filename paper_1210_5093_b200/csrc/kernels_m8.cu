// Match kernels (lanes, converge, ceiling) of table layout 8 (rep4_u8); see kernels.cu.
#define DFA_TU_MODE 8
#include "kernels.cu"
