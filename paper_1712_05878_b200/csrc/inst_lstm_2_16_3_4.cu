// kernel instantiations of lstm(2,16,3)→softmax(16,4) (inst.cuh)
#include "inst.cuh"
GHC_INST(2, 16, 3, 4)
