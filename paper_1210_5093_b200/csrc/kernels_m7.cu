// Match kernels (lanes, converge, ceiling) of table layout 7 (rep8_u8); see kernels.cu.
#define DFA_TU_MODE 7
#include "kernels.cu"
