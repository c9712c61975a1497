// fg_wm_p16.cu -- instantiations of the multi-row walk kernel for layout P16.
#include "fg_walk_multi.cuh"

cudaError_t fg_wm_p16(int ns, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (ns) {
    case 2: return fgwm::launch_wm<fgd::P16, 2>(a, num_sms, st);
    case 3: return fgwm::launch_wm<fgd::P16, 3>(a, num_sms, st);
    case 4: return fgwm::launch_wm<fgd::P16, 4>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
