// fg_verify.cu -- batched bit-sliced Brent verifier (reading R7)
// plus the small pool kernels (replicate seed, restart R23).
//
// verify_kernel: one CTA per queued scheme.  The scheme's 6 bit planes are staged
// in shared memory; thread t owns equation rows (a,b) (a over m*n, b over n*p) and
// accumulates sum_l u_l[a] v_l[b] w_l[.] over all c at once as an 11-plane
// bit-sliced two's-complement counter per c bit (r <= 512 < 2^10): per
// contributing term one ripple increment (positive w entries) and one ripple
// decrement (negative ones), 3 LOP3-class ops per plane.  The result must equal
// the matmul tensor slice T(a,b,.) = bit (k*m+i) iff a=i*n+j, b=j*p+k.  The
// lexicographically first failing (a,b,c) is an atomicMin over (a*np+b)*64+c.
#include "fg_device.cuh"

namespace {

constexpr int VTHREADS = 256;
constexpr int NPLANE = 11;

// One CTA checks one scheme (6 planes x R words at src, `rank` rows) against the
// Brent equations; returns ~0 if it verifies, else (a*np + b)*64 + c of the first
// failing equation (lexicographic).  sm: 6*R words of shared memory.
__device__ unsigned long long verify_scheme_cta(const uint64_t *src, int rank, int R, int m, int n, int p,
                                                int ring, uint64_t *sm, unsigned long long *first)
{
    const int mn = m * n, np = n * p, pm = p * m;
    const uint64_t cmask = pm == 64 ? ~0ull : ((1ull << pm) - 1ull);
    for (int t = threadIdx.x; t < FG_PLANES * R; t += blockDim.x) sm[t] = src[t];
    if (threadIdx.x == 0) *first = ~0ull;
    __syncthreads();
    for (int ab = threadIdx.x; ab < mn * np; ab += blockDim.x) {
        const int aa = ab / np, bb = ab - aa * np;
        uint64_t acc[NPLANE];
#pragma unroll
        for (int b = 0; b < NPLANE; ++b) acc[b] = 0;
        for (int l = 0; l < rank; ++l) {
            const uint64_t ud = sm[0 * R + l], vd = sm[2 * R + l];
            if (!(((ud >> aa) & (vd >> bb)) & 1ull)) continue;
            const uint64_t wd = sm[4 * R + l];
            if (ring == FG_Z2) { acc[0] ^= wd; continue; }
            const uint64_t ws = sm[5 * R + l];
            const uint64_t sn = (((sm[1 * R + l] >> aa) ^ (sm[3 * R + l] >> bb)) & 1ull) ? ~0ull : 0ull;
            uint64_t c = wd & ~(ws ^ sn);          // +1 entries
            uint64_t bo = wd & (ws ^ sn);          // -1 entries
#pragma unroll
            for (int b = 0; b < NPLANE; ++b) { const uint64_t t = acc[b] & c; acc[b] ^= c; c = t; }
#pragma unroll
            for (int b = 0; b < NPLANE; ++b) { const uint64_t t = ~acc[b] & bo; acc[b] ^= bo; bo = t; }
        }
        const int i = aa / n, j = aa - i * n, j2 = bb / p, k = bb - j2 * p;
        const uint64_t tm = (j == j2) ? (1ull << (k * m + i)) : 0ull;
        uint64_t mis = acc[0] ^ tm;
        if (ring == FG_ZT) {
#pragma unroll
            for (int b = 1; b < NPLANE; ++b) mis |= acc[b];
        }
        mis &= cmask;
        if (mis) atomicMin(first, ((unsigned long long)ab << 6) | (unsigned long long)(__ffsll((long long)mis) - 1));
    }
    __syncthreads();
    const unsigned long long res = *first;
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(VTHREADS) verify_kernel(VerifyArgs a)
{
    extern __shared__ uint64_t sm[];
    __shared__ unsigned long long first;
    const uint32_t count = a.count_ptr ? min(*a.count_ptr, a.cap) : a.count;
    const int np = a.n * a.p;
    for (uint32_t q = blockIdx.x; q < count; q += gridDim.x) {
        const unsigned long long f = verify_scheme_cta(a.planes + (size_t)q * FG_PLANES * a.R, a.meta[q].rank,
                                                       a.R, a.m, a.n, a.p, a.ring, sm, &first);
        if (threadIdx.x == 0) {
            fg_qmeta *qm = a.meta + q;
            if (f == ~0ull) {
                qm->ok = 1;
                qm->ff[0] = qm->ff[1] = qm->ff[2] = -1;
            } else {
                const int ab = (int)(f >> 6);
                qm->ok = 0;
                qm->ff[0] = ab / np;
                qm->ff[1] = ab % np;
                qm->ff[2] = (int)(f & 63);
                if (a.fail_count) atomicAdd(a.fail_count, 1u);
                if (a.hdr) atomicAdd((unsigned long long *)&a.hdr[qm->walker].cnt[FG_CNT_VERIFY_FAIL], 1ull);
            }
        }
    }
}

// Walkers whose strict improvements overflowed the queue (header flag bit 0):
// verify their final best scheme instead (the intermediate ones were never exported).
__global__ void __launch_bounds__(VTHREADS) verify_flagged_kernel(const uint64_t *best, fg_whdr *hdr, int64_t nwalk,
                                                                  int R, int m, int n, int p, int ring,
                                                                  uint32_t *fail_count, unsigned long long *done)
{
    extern __shared__ uint64_t sm[];
    __shared__ unsigned long long first;
    for (int64_t w = blockIdx.x; w < nwalk; w += gridDim.x) {
        if (!(hdr[w].pad & 1)) continue;
        const unsigned long long f = verify_scheme_cta(best + (size_t)w * FG_PLANES * R, hdr[w].best_r, R, m, n, p,
                                                       ring, sm, &first);
        if (threadIdx.x == 0) {
            hdr[w].pad &= ~1;
            atomicAdd(done, 1ull);
            if (f != ~0ull) {
                atomicAdd(fail_count, 1u);
                atomicAdd((unsigned long long *)&hdr[w].cnt[FG_CNT_VERIFY_FAIL], 1ull);
            }
        }
        __syncthreads();
    }
}

// R23: re-seed walkers whose best rank exceeds pool_rank + slack (one warp each)
__global__ void restart_kernel(uint64_t *cur, uint64_t *best, fg_whdr *hdr, int64_t nwalk, int R,
                               const uint64_t *pool, int pool_rank, int pool_adds, int slack,
                               unsigned long long *restarted)
{
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwalk; w += nw) {
        fg_whdr *h = hdr + w;
        if (!(h->best_r > pool_rank + slack)) continue;
        uint64_t *c = cur + (size_t)w * FG_PLANES * R, *b = best + (size_t)w * FG_PLANES * R;
        for (int t = lane; t < FG_PLANES * R; t += 32) { c[t] = pool[t]; b[t] = pool[t]; }
        __syncwarp();
        if (lane == 0) {
            h->r = pool_rank;
            h->best_r = pool_rank;
            h->best_adds = pool_adds;
            uint64_t d = (h->digest ^ (0xA5A5000000000000ULL | (uint64_t)(uint32_t)pool_rank)) * 0x100000001b3ULL;
            h->digest = d ^ (d >> 32);
            atomicAdd(restarted, 1ull);
        }
    }
}

// R20/R21 local best key over all walkers' best schemes (after seeding / restart /
// state load, and after a walk in which a verification failed; the walk kernels
// compute the same key in their epilogue)
__global__ void bestkey_kernel(const uint64_t *best, const fg_whdr *hdr, int64_t nwalk, int R, int mp,
                               unsigned long long *key)
{
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwalk; w += nw) {
        const int br = hdr[w].best_r;
        // unseeded walkers (rank 0) and walkers with a failed Brent check (R19) never
        // supply the best (whole warp takes the same branch)
        if (br < 1 || hdr[w].cnt[FG_CNT_VERIFY_FAIL] != 0) continue;
        const uint64_t *b = best + (size_t)w * FG_PLANES * R;
        int nnz = 0;
        for (int l = lane; l < br; l += 32)
            nnz += __popcll(b[0 * R + l]) + __popcll(b[2 * R + l]) + __popcll(b[4 * R + l]);
        nnz = __reduce_add_sync(0xffffffffu, nnz);
        if (lane == 0) {
            int adds = nnz - 2 * br - mp;
            if (adds < 0) adds = 0;
            atomicMin(key, ((unsigned long long)br << 54) | ((unsigned long long)adds << 36) |
                               (unsigned long long)w);
        }
    }
}

// Exact time-to-rank: the first step index at which a VERIFIED strict
// improvement reached each rank, from the verify queue entries of this launch.
__global__ void rank_first_kernel(const fg_qmeta *meta, const uint32_t *count_ptr, uint32_t cap,
                                  unsigned long long *first)
{
    const uint32_t count = min(*count_ptr, cap);
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x)
        if (meta[q].ok == 1 && meta[q].rank >= 0 && meta[q].rank <= FG_MAX_RCAP)
            atomicMin(first + meta[q].rank, (unsigned long long)meta[q].step);
}

}  // namespace

cudaError_t fg_launch_rank_first(const fg_qmeta *meta, const uint32_t *count_ptr, uint32_t cap,
                                 unsigned long long *first, cudaStream_t st)
{
    rank_first_kernel<<<64, 256, 0, st>>>(meta, count_ptr, cap, first);
    return cudaGetLastError();
}

cudaError_t fg_launch_bestkey(const uint64_t *best, const fg_whdr *hdr, int64_t num_walkers, int R, int mp,
                              unsigned long long *key, cudaStream_t st)
{
    int64_t blocks = (num_walkers * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    bestkey_kernel<<<(unsigned)blocks, 256, 0, st>>>(best, hdr, num_walkers, R, mp, key);
    return cudaGetLastError();
}

cudaError_t fg_launch_verify(const VerifyArgs &a, cudaStream_t st)
{
    const size_t smem = (size_t)FG_PLANES * a.R * sizeof(uint64_t);
    const uint32_t grid = a.count_ptr ? 2 * 148 * 4 : (a.count ? a.count : 1);
    verify_kernel<<<grid < 65535 ? grid : 65535, VTHREADS, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t fg_launch_verify_flagged(const uint64_t *best, fg_whdr *hdr, int64_t num_walkers, int R, int m,
                                     int n, int p, int ring, uint32_t *fail_count, unsigned long long *done,
                                     cudaStream_t st)
{
    const size_t smem = (size_t)FG_PLANES * R * sizeof(uint64_t);
    int64_t blocks = num_walkers < 148 * 8 ? num_walkers : 148 * 8;
    verify_flagged_kernel<<<(unsigned)blocks, VTHREADS, smem, st>>>(best, hdr, num_walkers, R, m, n, p, ring,
                                                                      fail_count, done);
    return cudaGetLastError();
}

cudaError_t fg_launch_restart(uint64_t *cur, uint64_t *best, fg_whdr *hdr, int64_t num_walkers,
                              int R, const uint64_t *pool_planes, int pool_rank, int pool_adds, int slack,
                              unsigned long long *restarted, cudaStream_t st)
{
    int64_t blocks = (num_walkers * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    restart_kernel<<<(unsigned)blocks, 256, 0, st>>>(cur, best, hdr, num_walkers, R, pool_planes,
                                                      pool_rank, pool_adds, slack, restarted);
    return cudaGetLastError();
}
