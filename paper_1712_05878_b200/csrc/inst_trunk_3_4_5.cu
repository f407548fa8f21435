// kernel instantiations of the LSTM trunk lstm(3,4,5) (inst.cuh)
#include "inst.cuh"
GHC_INST_TRUNK(3, 4, 5)
