#define SWB_X_T 2
#define SWB_X_GE 2
#define SWB_X_LO 33
#define SWB_X_HI 40
#define SWB_X_FILL swb_fill_exact_t2_g2_c
#include "sw_inst_exact.inc"
