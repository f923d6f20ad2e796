// Explicit instantiation of the fp32 engine (split from fp64 for parallel builds).
#include "engine_impl.cuh"
template class mfd::Engine<float>;
