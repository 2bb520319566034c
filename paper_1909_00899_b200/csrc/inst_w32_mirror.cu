#define SWB_INST_WORD W32
#define SWB_INST_VAR VAR_LAZYF_MIRROR
#define SWB_INST_FILL swb_fill_w32_mirror
#include "sw_inst.inc"
