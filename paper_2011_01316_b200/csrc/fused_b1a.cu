// Explicit instantiations of the fused small-problem engines (ctl.cuh) for collocated 1D Burgers, in
// their own translation unit so the build compiles them in parallel.
#include "ctl.cuh"

namespace expdg {

template void launch_phi_fused<B1FusedElem<2>>(cudaStream_t, Engine&, const B1FusedElem<2>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<3>>(cudaStream_t, Engine&, const B1FusedElem<3>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<4>>(cudaStream_t, Engine&, const B1FusedElem<4>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<5>>(cudaStream_t, Engine&, const B1FusedElem<5>&, const BArgs&);

}  // namespace expdg
