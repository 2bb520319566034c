#define SWB_INST_WORD W16
#define SWB_INST_VAR VAR_LAZYF_MIRROR
#define SWB_INST_FILL swb_fill_w16_mirror
#include "sw_inst.inc"
