// Match kernels (lanes, converge, ceiling) of table layout 2 (ident_u16); see kernels.cu.
#define DFA_TU_MODE 2
#include "kernels.cu"
