#define SWB_X_T 4
#define SWB_X_GE 1
#define SWB_X_LO 57
#define SWB_X_HI 64
#define SWB_X_FILL swb_fill_exact_t4_g1_f
#include "sw_inst_exact.inc"
