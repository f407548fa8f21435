// kernel instantiations of the LSTM trunk lstm(5,8,10) (inst.cuh)
#include "inst.cuh"
GHC_INST_TRUNK(5, 8, 10)
