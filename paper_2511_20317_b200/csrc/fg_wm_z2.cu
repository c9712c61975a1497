// fg_wm_z2.cu -- instantiations of the multi-row walk kernel for layout PZ2.
#include "fg_walk_multi.cuh"

cudaError_t fg_wm_z2(int ns, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (ns) {
    case 2: return fgwm::launch_wm<fgd::PZ2, 2>(a, num_sms, st);
    case 3: return fgwm::launch_wm<fgd::PZ2, 3>(a, num_sms, st);
    case 4: return fgwm::launch_wm<fgd::PZ2, 4>(a, num_sms, st);
    case 5: return fgwm::launch_wm<fgd::PZ2, 5>(a, num_sms, st);
    case 6: return fgwm::launch_wm<fgd::PZ2, 6>(a, num_sms, st);
    case 8: return fgwm::launch_wm<fgd::PZ2, 8>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
