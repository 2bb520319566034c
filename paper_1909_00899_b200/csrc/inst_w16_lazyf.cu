#define SWB_INST_WORD W16
#define SWB_INST_VAR VAR_LAZYF
#define SWB_INST_FILL swb_fill_w16_lazyf
#include "sw_inst.inc"
