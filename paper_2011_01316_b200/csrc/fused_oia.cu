// Explicit instantiations of the fused small-problem engines (ctl.cuh) for over-integrated 1D Burgers, in
// their own translation unit so the build compiles them in parallel.
#include "ctl.cuh"

namespace expdg {

#define FUSED_OI(NP, NQ) \
  template void launch_phi_fused<B1OIFusedElem<NP, NQ>>(cudaStream_t, Engine&, const B1OIFusedElem<NP, NQ>&, \
                                                        const BArgs&);
FUSED_OI(2, 3)
FUSED_OI(3, 4)
FUSED_OI(4, 6)
FUSED_OI(5, 7)
#undef FUSED_OI

}  // namespace expdg
