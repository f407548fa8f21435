// kernel instantiations of the LSTM trunk lstm(5,20,10) (inst.cuh)
#include "inst.cuh"
GHC_INST_TRUNK(5, 20, 10)
