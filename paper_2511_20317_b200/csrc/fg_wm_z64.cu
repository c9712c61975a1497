// fg_wm_z64.cu -- instantiations of the multi-row walk kernel for layout PZ64.
#include "fg_walk_multi.cuh"

cudaError_t fg_wm_z64(int ns, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (ns) {
    case 4: return fgwm::launch_wm<fgd::PZ64, 4>(a, num_sms, st);
    case 6: return fgwm::launch_wm<fgd::PZ64, 6>(a, num_sms, st);
    case 8: return fgwm::launch_wm<fgd::PZ64, 8>(a, num_sms, st);
    case 10: return fgwm::launch_wm<fgd::PZ64, 10>(a, num_sms, st);
    case 13: return fgwm::launch_wm<fgd::PZ64, 13>(a, num_sms, st);
    case 16: return fgwm::launch_wm<fgd::PZ64, 16>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
