// Explicit instantiation of the fp32 engine (split from fp64 for parallel builds).
#include "engine_impl.cuh"
#include "virtual_group.cuh"
template class mfd::Engine<float>;
template class mfd::VirtualGroup<float>;
namespace mfd {
template <>
EngineBase* make_engine<float>(const mfd_grid& g, const mfd_material& m, const mfd_terms& te, const mfd_stepper& st,
                               int device, int rank, int world, Transport* tr) {
    return new Engine<float>(g, m, te, st, device, Slab::of(g.nz, rank, world), tr);
}
template <>
EngineBase* make_virtual_group<float>(const mfd_grid& g, const mfd_material& m, const mfd_terms& te,
                                      const mfd_stepper& st, int device, int world) {
    return new VirtualGroup<float>(g, m, te, st, device, world);
}
} // namespace mfd
