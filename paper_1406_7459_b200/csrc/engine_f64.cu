// Explicit instantiation of the fp64 engine (split from fp32 for parallel builds).
#include "engine_impl.cuh"
#include "virtual_group.cuh"
template class mfd::Engine<double>;
template class mfd::VirtualGroup<double>;
namespace mfd {
template <>
EngineBase* make_engine<double>(const mfd_grid& g, const mfd_material& m, const mfd_terms& te, const mfd_stepper& st,
                               int device, int rank, int world, Transport* tr) {
    return new Engine<double>(g, m, te, st, device, Slab::of(g.nz, rank, world), tr);
}
template <>
EngineBase* make_virtual_group<double>(const mfd_grid& g, const mfd_material& m, const mfd_terms& te,
                                      const mfd_stepper& st, int device, int world) {
    return new VirtualGroup<double>(g, m, te, st, device, world);
}
} // namespace mfd
