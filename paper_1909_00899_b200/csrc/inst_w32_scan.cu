#define SWB_INST_WORD W32
#define SWB_INST_VAR VAR_SCAN
#define SWB_INST_FILL swb_fill_w32_scan
#include "sw_inst.inc"
