// kernel instantiations of lstm(5,8,10)→softmax(8,3) (inst.cuh)
#include "inst.cuh"
GHC_INST(5, 8, 10, 3)
