#include "../pass_instantiate.cuh"
LATTDSE_INSTANTIATE_L(2160)
