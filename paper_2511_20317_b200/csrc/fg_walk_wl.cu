// fg_walk_wl.cu -- dispatch of the linked-class one-walker-per-warp kernel
// (fg_walk_wl.cuh) over the factor layouts.
#include "fg_walk_wl.cuh"

using namespace fgd;

size_t fg_wl_img_words(int R) { return (size_t)fgwl::img_words((R + 31) / 32); }

bool fg_kind_is_wl(int kind)
{
    return kind == FG_K_WL_P16 || kind == FG_K_WL_P32 || kind == FG_K_WL_P64 || kind == FG_K_WL_Z2 ||
           kind == FG_K_WL_Z64;
}

cudaError_t fg_launch_walk_wl(int kind, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (kind) {
    case FG_K_WL_P16: return fgwl::launch_wl<P16>(a, num_sms, st);
    case FG_K_WL_P32: return fgwl::launch_wl<P32>(a, num_sms, st);
    case FG_K_WL_P64: return fgwl::launch_wl<P64>(a, num_sms, st);
    case FG_K_WL_Z2: return fgwl::launch_wl<PZ2>(a, num_sms, st);
    case FG_K_WL_Z64: return fgwl::launch_wl<PZ64>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
