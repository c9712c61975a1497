// fg_internal.h -- private types shared by libfg's host code and kernels.
// Nothing here is part of the ABI (include/fg.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/fg.h"

// Device layout of one scheme: 6 bit planes x R rows of u64 words, plane-major:
//   plane 0 u.digits, 1 u.signs, 2 v.digits, 3 v.signs, 4 w.digits, 5 w.signs
// ("one-bit representation"; Z_2 leaves the sign planes 0).
// Walker k's scheme starts at k*6*R; a warp reads plane q of rows 0..31 as 32
// consecutive u64 (256 B, coalesced).
#define FG_PLANES 6

struct __align__(16) fg_whdr {     // per-walker header, 128 B
    int32_t r;
    int32_t best_r;
    uint64_t step;                 // Alg.1 iteration index since seeding (R8)
    uint64_t digest;
    uint64_t cnt[FG_NCNT];
    int32_t best_adds;             // naive additions of the best scheme
    int32_t pad;                   // bit 0: a strict improvement missed the verify queue
};
static_assert(sizeof(fg_whdr) == 128, "fg_whdr size");

struct fg_qmeta {                  // one verify-queue entry
    int64_t walker;                // local walker index
    uint64_t step;                 // step index at which it was found
    int32_t rank;
    int32_t ok;                    // filled by the verifier: 1 pass, 0 fail
    int32_t ff[3];                 // first failing (a,b,c) or -1
    int32_t pad;
};

enum { FG_CNT_STEPS = 0, FG_CNT_DRAWS, FG_CNT_FLIPS, FG_CNT_FLIP_FAIL, FG_CNT_EXPAND_OK,
       FG_CNT_EXPAND_REJECT, FG_CNT_MERGES, FG_CNT_ZERO_REMOVED, FG_CNT_BEST_COPIES,
       FG_CNT_IMPROVEMENTS, FG_CNT_REDUCE_CALLS, FG_CNT_VERIFY_FAIL };

struct WalkArgs {
    uint64_t *cur;
    uint64_t *best;
    fg_whdr *hdr;
    int64_t num_walkers;
    int64_t id_base;
    int m, n, p, R;
    int len_u, len_v, len_w;
    int mp;
    uint64_t steps;
    uint64_t seed;
    uint32_t k_flip, thr_eq, thr_reduce, thr_expand;
    int32_t slack;
    // verify queue (strict improvements, R19)
    uint64_t *q_planes;
    fg_qmeta *q_meta;
    uint32_t *q_count;
    uint32_t q_cap;
    uint32_t *q_overflow;
    // local best key (R20): rank<<54 | additions<<36 | local walker index
    unsigned long long *best_key;
    unsigned long long *work_counter;   // dynamic walker queue, zeroed before each launch
    uint32_t *task_done;                // walk_ql: per walker group, chunks stored (zeroed per launch)
    uint32_t chunks;                    // walk_ql: step chunks per group (set by its launcher)
    uint64_t chunk_steps;
    uint32_t *ql_img;                   // walk_ql / walk_q4: per-walker shared-memory image between chunks
    uint32_t *ring;                     // walk_q4: ready queue of groups (group+1 per slot, zeroed per launch)
    unsigned long long *ring_tail;      // walk_q4: completed chunks so far (zeroed per launch)
    uint32_t *wl_img;                   // walk_wl: per-walker class image (links, later counts) between launches
    uint32_t img_valid;                 // walk_wl: wl_img matches the walkers' current rows
    uint32_t mode;                      // 0 = Alg. 1 walk, 1 = naive-complexity minimisation (R24)
    uint32_t dbg;                       // debug switches (env FG_DBG), 0 in production
    uint32_t *dbgbuf;                   // 16 words of debug output (first error wins)
};

struct VerifyArgs {
    const uint64_t *planes;        // count schemes, 6*R u64 each
    fg_qmeta *meta;                // rank in, ok/ff out
    const uint32_t *count_ptr;     // device count (queue) or nullptr -> count
    uint32_t count;
    uint32_t cap;
    int m, n, p, R, ring;
    fg_whdr *hdr;                  // if non-null: failures bump hdr[walker].cnt[VERIFY_FAIL]
    uint32_t *fail_count;
};

// launchers (fg_walk.cu / fg_verify.cu); return cudaError_t
enum fg_kernel_kind { FG_K_NONE = 0, FG_K_W32_ZT_K16, FG_K_W32_ZT_K32, FG_K_W32_Z2_K32,
                      FG_K_WM_P16, FG_K_WM_P32, FG_K_WM_P64, FG_K_WM_Z2, FG_K_WM_Z64,
                      FG_K_Q4_P16, FG_K_Q4_Z2, FG_K_QL_P16, FG_K_QL_Z2,
                      FG_K_WL_P16, FG_K_WL_P32, FG_K_WL_P64, FG_K_WL_Z2, FG_K_WL_Z64 };
cudaError_t fg_launch_walk_wl(int kind, const WalkArgs &a, int num_sms, cudaStream_t st);
size_t fg_wl_img_words(int R);     // walk_wl class image words per walker
bool fg_kind_is_wl(int kind);
cudaError_t fg_launch_walk_ql(int kind, const WalkArgs &a, int num_sms, cudaStream_t st);
cudaError_t fg_launch_walk_q4(int kind, const WalkArgs &a, int num_sms, cudaStream_t st);
int fg_multi_ns(int R);
int fg_multi_kind(int ring, int maxlen, int R);
cudaError_t fg_launch_walk_multi(int kind, int ns, const WalkArgs &a, int num_sms, cudaStream_t st);
int fg_pick_kernel(int ring, int maxlen, int R);
const char *fg_kernel_kind_name(int kind);
cudaError_t fg_launch_walk(int kind, const WalkArgs &a, int num_sms, cudaStream_t st);
cudaError_t fg_launch_verify(const VerifyArgs &a, cudaStream_t st);
cudaError_t fg_launch_restart(uint64_t *cur, uint64_t *best, fg_whdr *hdr, int64_t num_walkers,
                              int R, const uint64_t *pool_planes, int pool_rank, int pool_adds, int slack,
                              unsigned long long *restarted, cudaStream_t st);
int fg_kind_for_mode(int kind);
cudaError_t fg_launch_verify_flagged(const uint64_t *best, fg_whdr *hdr, int64_t num_walkers, int R, int m,
                                     int n, int p, int ring, uint32_t *fail_count, unsigned long long *done,
                                     cudaStream_t st);   // R24 runs on the quad, one-walker-per-warp and multi-row kernels
cudaError_t fg_launch_rank_first(const fg_qmeta *meta, const uint32_t *count_ptr, uint32_t cap,
                                 unsigned long long *first, cudaStream_t st);
cudaError_t fg_launch_bestkey(const uint64_t *best, const fg_whdr *hdr, int64_t num_walkers, int R, int mp,
                              unsigned long long *key, cudaStream_t st);
