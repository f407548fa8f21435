// kernel instantiations of lstm(5,20,10)→softmax(20,3) (inst.cuh)
#include "inst.cuh"
GHC_INST(5, 20, 10, 3)
