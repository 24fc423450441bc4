// Single translation unit for libpipeplan_b200.so.
#include "prm.cu"
#include "rdo.cu"
#include "dp_persist.cu"
#include "dp_inst.cu"
#include "sim.cu"
#include "capi.cu"
#include "trace.cu"
#include "validate.cu"
