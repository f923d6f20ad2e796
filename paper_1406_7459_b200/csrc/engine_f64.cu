// Explicit instantiation of the fp64 engine (split from fp32 for parallel builds).
#include "engine_impl.cuh"
template class mfd::Engine<double>;
