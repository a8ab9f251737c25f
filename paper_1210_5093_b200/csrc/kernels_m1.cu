// Match kernels (lanes, converge, ceiling) of table layout 1 (ident_u8); see kernels.cu.
#define DFA_TU_MODE 1
#include "kernels.cu"
