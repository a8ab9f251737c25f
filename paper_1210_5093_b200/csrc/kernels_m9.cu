// Match kernels (lanes, converge, ceiling) of table layout 9 (ident_u8_pad); see kernels.cu.
#define DFA_TU_MODE 9
#include "kernels.cu"
