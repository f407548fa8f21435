// kernel instantiations of lstm(4,12,6)→softmax(12,5) (inst.cuh)
#include "inst.cuh"
GHC_INST(4, 12, 6, 5)
