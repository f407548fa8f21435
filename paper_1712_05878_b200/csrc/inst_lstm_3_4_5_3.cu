// kernel instantiations of lstm(3,4,5)→softmax(4,3) (inst.cuh)
#include "inst.cuh"
GHC_INST(3, 4, 5, 3)
