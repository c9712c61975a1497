// fg_walk_multi.cu -- dispatch of the multi-row walk kernel (fg_walk_multi.cuh) over
// factor layouts and slots per lane; each layout is instantiated in its own
// translation unit (fg_wm_<policy>.cu) so the build compiles them in parallel.
#include "fg_internal.h"

cudaError_t fg_wm_p16(int ns, const WalkArgs &a, int num_sms, cudaStream_t st);
cudaError_t fg_wm_p32(int ns, const WalkArgs &a, int num_sms, cudaStream_t st);
cudaError_t fg_wm_p64(int ns, const WalkArgs &a, int num_sms, cudaStream_t st);
cudaError_t fg_wm_z2(int ns, const WalkArgs &a, int num_sms, cudaStream_t st);
cudaError_t fg_wm_z64(int ns, const WalkArgs &a, int num_sms, cudaStream_t st);

// slots per lane available per layout (R up to 32*NS)
static const int NS_P16[] = {2, 3, 4};
static const int NS_P32[] = {2, 3, 4, 5, 6, 8};
static const int NS_P64[] = {4, 6, 8, 10, 13, 16};

static int pick(const int *list, int n, int R)
{
    for (int k = 0; k < n; ++k)
        if (32 * list[k] >= R) return list[k];
    return 0;
}

int fg_multi_ns(int R) { return pick(NS_P64, 6, R); }

// narrowest layout that holds the factors and has a slot count for R
int fg_multi_kind(int ring, int maxlen, int R)
{
    if (R > 512) return FG_K_NONE;
    if (ring == FG_ZT) {
        if (maxlen <= 16 && pick(NS_P16, 3, R)) return FG_K_WM_P16;
        if (maxlen <= 32 && pick(NS_P32, 6, R)) return FG_K_WM_P32;
        return FG_K_WM_P64;
    }
    if (maxlen <= 32 && pick(NS_P32, 6, R)) return FG_K_WM_Z2;
    return FG_K_WM_Z64;
}

cudaError_t fg_launch_walk_multi(int kind, int, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (kind) {
    case FG_K_WM_P16: return fg_wm_p16(pick(NS_P16, 3, a.R), a, num_sms, st);
    case FG_K_WM_P32: return fg_wm_p32(pick(NS_P32, 6, a.R), a, num_sms, st);
    case FG_K_WM_P64: return fg_wm_p64(pick(NS_P64, 6, a.R), a, num_sms, st);
    case FG_K_WM_Z2: return fg_wm_z2(pick(NS_P32, 6, a.R), a, num_sms, st);
    case FG_K_WM_Z64: return fg_wm_z64(pick(NS_P64, 6, a.R), a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
