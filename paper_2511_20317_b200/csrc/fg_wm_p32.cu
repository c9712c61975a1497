// fg_wm_p32.cu -- instantiations of the multi-row walk kernel for layout P32.
#include "fg_walk_multi.cuh"

cudaError_t fg_wm_p32(int ns, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (ns) {
    case 2: return fgwm::launch_wm<fgd::P32, 2>(a, num_sms, st);
    case 3: return fgwm::launch_wm<fgd::P32, 3>(a, num_sms, st);
    case 4: return fgwm::launch_wm<fgd::P32, 4>(a, num_sms, st);
    case 5: return fgwm::launch_wm<fgd::P32, 5>(a, num_sms, st);
    case 6: return fgwm::launch_wm<fgd::P32, 6>(a, num_sms, st);
    case 8: return fgwm::launch_wm<fgd::P32, 8>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
