// Match kernels (lanes, converge, ceiling) of table layout 5 (packed9); see kernels.cu.
#define DFA_TU_MODE 5
#include "kernels.cu"
