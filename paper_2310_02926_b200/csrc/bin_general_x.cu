// bin_general_x.cu -- the BIN_SUM_EXACT instances of the general accumulate
// kernel (bin_general.cu compiled with BIN_GENERAL_XS = 1; a separate
// translation unit so the two instance sets compile in parallel).
#define BIN_GENERAL_XS 1
#include "bin_general.cu"
