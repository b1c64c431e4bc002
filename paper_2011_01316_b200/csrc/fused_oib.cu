// Explicit instantiations of the fused small-problem engines (ctl.cuh) for over-integrated 1D Burgers, in
// their own translation unit so the build compiles them in parallel.
#include "ctl.cuh"

namespace expdg {

#define FUSED_OI(NP, NQ) \
  template void launch_phi_fused<B1OIFusedElem<NP, NQ>>(cudaStream_t, Engine&, const B1OIFusedElem<NP, NQ>&, \
                                                        const BArgs&);
FUSED_OI(6, 9)
FUSED_OI(7, 10)
FUSED_OI(8, 12)
FUSED_OI(9, 13)
#undef FUSED_OI

}  // namespace expdg
