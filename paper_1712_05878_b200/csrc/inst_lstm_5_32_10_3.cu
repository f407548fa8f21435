// kernel instantiations of lstm(5,32,10)→softmax(32,3) (inst.cuh)
#include "inst.cuh"
GHC_INST(5, 32, 10, 3)
