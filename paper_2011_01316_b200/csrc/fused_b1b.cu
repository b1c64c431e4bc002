// Explicit instantiations of the fused small-problem engines (ctl.cuh) for collocated 1D Burgers, in
// their own translation unit so the build compiles them in parallel.
#include "ctl.cuh"

namespace expdg {

template void launch_phi_fused<B1FusedElem<6>>(cudaStream_t, Engine&, const B1FusedElem<6>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<7>>(cudaStream_t, Engine&, const B1FusedElem<7>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<8>>(cudaStream_t, Engine&, const B1FusedElem<8>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<9>>(cudaStream_t, Engine&, const B1FusedElem<9>&, const BArgs&);

}  // namespace expdg
