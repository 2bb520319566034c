#define SWB_X_T 4
#define SWB_X_GE 1
#define SWB_X_LO 41
#define SWB_X_HI 48
#define SWB_X_FILL swb_fill_exact_t4_g1_d
#include "sw_inst_exact.inc"
