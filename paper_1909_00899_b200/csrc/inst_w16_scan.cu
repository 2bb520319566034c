#define SWB_INST_WORD W16
#define SWB_INST_VAR VAR_SCAN
#define SWB_INST_FILL swb_fill_w16_scan
#include "sw_inst.inc"
