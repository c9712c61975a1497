// fg_host.cu -- host side of libfg.so: the C ABI of include/fg.h.
// Owns device memory, packs int8 schemes into bit planes, launches the walk /
// verify / restart kernels on the caller's stream, keeps the local + pool best.
// No torch types; no dependency on oracle/.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>
#include "fg_internal.h"

namespace {

constexpr uint32_t REC_MAGIC = 0x46475231u;   // "FGR1"
constexpr uint32_t STATE_MAGIC = 0x46475333u; // "FGS3": packed planes; walk_wl word totals as 3 x 21-bit fields

struct RecHdr {          // 64 bytes, followed by 6*r_cap u64 planes
    uint32_t magic;
    int32_t m, n, p, ring, r_cap, rank, additions;
    int64_t walker_id;
    int32_t valid;
    int32_t pad[5];
};
static_assert(sizeof(RecHdr) == 64, "RecHdr size");

struct DevMisc {         // small device-side scratch read back after every fg_walk
    unsigned long long best_key;
    uint32_t q_count;
    uint32_t q_overflow;
    uint32_t verify_fail;
    uint32_t pad;
    unsigned long long restarted;
    unsigned long long work_counter;
    unsigned long long ring_tail;
    uint32_t dbgbuf[16];
};

}  // namespace

struct fg_ctx {
    int m, n, p, ring, R, maxlen, kind;
    int len[3];
    int64_t W, id_base;
    int device, num_sms;
    cudaStream_t stream;
    bool seeded;                       // every walker in [0, W) holds a scheme
    std::vector<std::pair<int64_t, int64_t>> covered;   // seeded walker ranges, merged
    // device
    uint64_t *d_cur, *d_best, *d_qplanes, *d_pool;
    fg_whdr *d_hdr;
    fg_qmeta *d_qmeta;
    DevMisc *d_misc;
    uint32_t *d_task_done;   // walk_ql chunk flags, one per walker group of 8
    uint32_t *d_ql_img;      // walk_ql / walk_q4: shared-memory image per walker between chunks
    uint32_t *d_ring;        // walk_q4: ready queue of step-chunk tasks
    uint32_t *d_wl_img;      // walk_wl: class image per walker between launches
    void *d_stage = nullptr; // fg_save_state / fg_load_state: packed planes (lazily allocated)
    unsigned long long *d_rank_first;   // [FG_MAX_RCAP + 1]: first step of a verified improvement to each rank
    bool img_valid;          // d_wl_img matches the walkers' rows (cleared by every host write)
    uint32_t qcap;
    cudaEvent_t ev0, ev1, ev2;
    // host bests
    std::vector<unsigned char> local_rec, pool_rec;
    // stats
    uint64_t st_steps, st_draws, st_flips, st_expands, st_reductions, st_verified, st_vfail,
        st_overflow, st_launches, st_walk_us, st_verify_us, st_walk_launches;
};

namespace {

int cuda_err(cudaError_t e)
{
    if (e == cudaSuccess) return FG_OK;
    fprintf(stderr, "libfg: CUDA error %d (%s)\n", (int)e, cudaGetErrorString(e));
    return FG_E_CUDA;
}

#define CK(x)                                   \
    do {                                        \
        int _rc = cuda_err(x);                  \
        if (_rc != FG_OK) return _rc;           \
    } while (0)

int width_of(int m, int n, int p) { return m * n + n * p + p * m; }

bool format_ok(int m, int n, int p)
{
    return m >= 1 && n >= 1 && p >= 1 && m * n <= FG_MAX_LEN && n * p <= FG_MAX_LEN &&
           p * m <= FG_MAX_LEN;
}

// int8 rows (interchange layout) -> 6 planes x R words; returns FG_E_DOMAIN on a
// coefficient outside the ring.
int pack_planes(int m, int n, int p, int ring, const int8_t *coeffs, int rank, int R, uint64_t *planes)
{
    const int len[3] = {m * n, n * p, p * m};
    const int w = len[0] + len[1] + len[2];
    std::fill(planes, planes + (size_t)FG_PLANES * R, 0ull);
    for (int l = 0; l < rank; ++l) {
        const int8_t *row = coeffs + (size_t)l * w;
        int off = 0;
        for (int X = 0; X < 3; ++X) {
            uint64_t d = 0, s = 0;
            for (int e = 0; e < len[X]; ++e) {
                const int v = row[off + e];
                if (v == 0) continue;
                if (v == 1) d |= 1ull << e;
                else if (v == -1 && ring == FG_ZT) { d |= 1ull << e; s |= 1ull << e; }
                else return FG_E_DOMAIN;
            }
            planes[(2 * X) * R + l] = d;
            planes[(2 * X + 1) * R + l] = s;
            off += len[X];
        }
    }
    return FG_OK;
}

void unpack_planes(int m, int n, int p, const uint64_t *planes, int R, int rank, int8_t *coeffs)
{
    const int len[3] = {m * n, n * p, p * m};
    const int w = len[0] + len[1] + len[2];
    for (int l = 0; l < rank; ++l) {
        int8_t *row = coeffs + (size_t)l * w;
        int off = 0;
        for (int X = 0; X < 3; ++X) {
            const uint64_t d = planes[(2 * X) * R + l], s = planes[(2 * X + 1) * R + l];
            for (int e = 0; e < len[X]; ++e)
                row[off + e] = ((d >> e) & 1) ? (((s >> e) & 1) ? -1 : 1) : 0;
            off += len[X];
        }
    }
}

// PAPER:429 per row on planes (R6)
void normalize_planes(uint64_t *planes, int R, int rank)
{
    for (int l = 0; l < rank; ++l) {
        uint64_t &ud = planes[0 * R + l], &us = planes[1 * R + l];
        uint64_t &vd = planes[2 * R + l], &vs = planes[3 * R + l];
        uint64_t &wd = planes[4 * R + l], &ws = planes[5 * R + l];
        if (us & (ud & (0 - ud))) { us ^= ud; ws ^= wd; }
        if (vs & (vd & (0 - vd))) { vs ^= vd; ws ^= wd; }
    }
}

int additions_planes(int m, int p, const uint64_t *planes, int R, int rank)
{
    int nnz = 0;
    for (int l = 0; l < rank; ++l)
        nnz += __builtin_popcountll(planes[0 * R + l]) + __builtin_popcountll(planes[2 * R + l]) +
               __builtin_popcountll(planes[4 * R + l]);
    return nnz - 2 * rank - m * p;
}

// Host Brent check on planes: accumulate the scheme tensor slice by slice
// (sparse over the nonzeros of u_l and v_l) and compare with T.
int verify_planes(int m, int n, int p, int ring, const uint64_t *planes, int R, int rank, int32_t ff[3])
{
    const int mn = m * n, np = n * p, pm = p * m;
    std::vector<int32_t> acc((size_t)mn * np * pm, 0);
    for (int l = 0; l < rank; ++l) {
        const uint64_t ud = planes[0 * R + l], us = planes[1 * R + l];
        const uint64_t vd = planes[2 * R + l], vs = planes[3 * R + l];
        const uint64_t wd = planes[4 * R + l], ws = planes[5 * R + l];
        for (uint64_t ua = ud; ua; ua &= ua - 1) {
            const int a = __builtin_ctzll(ua);
            const int sa = (us >> a) & 1;
            for (uint64_t vb = vd; vb; vb &= vb - 1) {
                const int b = __builtin_ctzll(vb);
                const int sab = sa ^ ((vs >> b) & 1);
                int32_t *slot = &acc[((size_t)a * np + b) * pm];
                for (uint64_t wc = wd; wc; wc &= wc - 1) {
                    const int c = __builtin_ctzll(wc);
                    slot[c] += (sab ^ ((ws >> c) & 1)) ? -1 : 1;
                }
            }
        }
    }
    for (int a = 0; a < mn; ++a)
        for (int b = 0; b < np; ++b)
            for (int c = 0; c < pm; ++c) {
                const int i = a / n, j = a % n, j2 = b / p, k = b % p, k2 = c / m, i2 = c % m;
                const int t = (j == j2 && k == k2 && i == i2) ? 1 : 0;
                int v = acc[((size_t)a * np + b) * pm + c];
                if (ring == FG_Z2) v &= 1;
                if (v != t) {
                    if (ff) { ff[0] = a; ff[1] = b; ff[2] = c; }
                    return FG_E_INVALID_SCHEME;
                }
            }
    if (ff) ff[0] = ff[1] = ff[2] = -1;
    return FG_OK;
}

bool has_zero_factor(const uint64_t *planes, int R, int rank)
{
    for (int l = 0; l < rank; ++l)
        if (!planes[0 * R + l] || !planes[2 * R + l] || !planes[4 * R + l]) return true;
    return false;
}

size_t rec_bytes(int R) { return sizeof(RecHdr) + (size_t)FG_PLANES * R * sizeof(uint64_t); }

// R20: lexicographic (rank, additions, walker id); invalid records lose
bool rec_better(const RecHdr *a, const RecHdr *b)
{
    if (!b->valid) return a->valid;
    if (!a->valid) return false;
    if (a->rank != b->rank) return a->rank < b->rank;
    if (a->additions != b->additions) return a->additions < b->additions;
    return a->walker_id < b->walker_id;
}

__global__ void replicate_kernel(uint64_t *dst, const uint64_t *src, int64_t words, int64_t copies)
{
    const int64_t total = words * copies;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = src[t % words];
}

int replicate(fg_ctx *c, uint64_t *dst, const uint64_t *src_dev, int64_t words, int64_t copies)
{
    if (copies <= 0) return FG_OK;
    int64_t blocks = (words * copies + 255) / 256;
    if (blocks > (int64_t)c->num_sms * 32) blocks = (int64_t)c->num_sms * 32;
    replicate_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(dst, src_dev, words, copies);
    c->st_launches++;
    CK(cudaGetLastError());
    return FG_OK;
}

int recompute_local_best(fg_ctx *c);
int refresh_local_best(fg_ctx *c, unsigned long long key, bool reset);

// time-to-rank table: nothing reached yet except the seeded rank, at step 0
int reset_rank_first(fg_ctx *c, int seeded_rank)
{
    std::vector<unsigned long long> v(FG_MAX_RCAP + 1, ~0ull);
    if (seeded_rank >= 0 && seeded_rank <= FG_MAX_RCAP) v[seeded_rank] = 0;
    CK(cudaMemcpyAsync(c->d_rank_first, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FG_OK;
}

// record [w0, w1) as seeded; the ctx is walkable once the ranges cover [0, W)
void mark_covered(fg_ctx *c, int64_t w0, int64_t w1)
{
    auto &v = c->covered;
    v.push_back({w0, w1});
    std::sort(v.begin(), v.end());
    std::vector<std::pair<int64_t, int64_t>> out;
    for (const auto &x : v) {
        if (!out.empty() && x.first <= out.back().second) out.back().second = std::max(out.back().second, x.second);
        else out.push_back(x);
    }
    v.swap(out);
    c->seeded = v.size() == 1 && v[0].first == 0 && v[0].second == c->W;
}

int seed_planes(fg_ctx *c, const uint64_t *planes, int rank, int64_t w0, int64_t w1)
{
    const int64_t words = (int64_t)FG_PLANES * c->R;
    fg_whdr h;
    memset(&h, 0, sizeof(h));
    h.r = rank;
    h.best_r = rank;
    h.step = 0;
    h.digest = 0xcbf29ce484222325ULL;
    h.best_adds = additions_planes(c->m, c->p, planes, c->R, rank);
    uint64_t *tmp = nullptr;
    fg_whdr *tmph = nullptr;
    CK(cudaMallocAsync((void **)&tmp, words * sizeof(uint64_t), c->stream));
    CK(cudaMallocAsync((void **)&tmph, sizeof(fg_whdr), c->stream));
    CK(cudaMemcpyAsync(tmp, planes, words * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(tmph, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
    int rc = replicate(c, c->d_cur + w0 * words, tmp, words, w1 - w0);
    if (rc == FG_OK) rc = replicate(c, c->d_best + w0 * words, tmp, words, w1 - w0);
    if (rc == FG_OK)
        rc = replicate(c, (uint64_t *)(c->d_hdr + w0), (const uint64_t *)tmph,
                       sizeof(fg_whdr) / sizeof(uint64_t), w1 - w0);
    CK(cudaFreeAsync(tmp, c->stream));
    CK(cudaFreeAsync(tmph, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (rc != FG_OK) return rc;
    mark_covered(c, w0, w1);
    c->img_valid = false;
    if (c->seeded) {
        int rr = reset_rank_first(c, rank);
        if (rr != FG_OK) return rr;
    }
    // the local best is defined once every walker holds a scheme (a partial
    // seed must not let zeroed headers of unseeded walkers into the best key)
    return c->seeded ? recompute_local_best(c) : FG_OK;
}

// best key over the walkers' best schemes on the device, skipping walkers whose
// verification failed (bestkey_kernel)
int device_best_key(fg_ctx *c, unsigned long long *key)
{
    CK(cudaMemsetAsync(&c->d_misc->best_key, 0xff, sizeof(unsigned long long), c->stream));
    CK(fg_launch_bestkey(c->d_best, c->d_hdr, c->W, c->R, c->m * c->p, &c->d_misc->best_key, c->stream));
    c->st_launches++;
    *key = ~0ull;
    CK(cudaMemcpyAsync(key, &c->d_misc->best_key, sizeof(*key), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FG_OK;
}

// Build the record of the walker the key names and make it the local best if it is
// better (R20), or unconditionally with `reset` (seed / load / restart).  The record
// is checked against the Brent equations first (R19: an unverified scheme is never
// stored): a failure returns FG_E_INVALID_SCHEME and leaves the local best alone.
int refresh_local_best(fg_ctx *c, unsigned long long key, bool reset)
{
    const int64_t words = (int64_t)FG_PLANES * c->R;
    const int64_t wk = (int64_t)(key & ((1ull << 36) - 1));
    if (reset) ((RecHdr *)c->local_rec.data())->valid = 0;
    if (key == ~0ull || wk >= c->W) return FG_OK;
    std::vector<unsigned char> cand(rec_bytes(c->R), 0);
    RecHdr *ch = (RecHdr *)cand.data();
    uint64_t *pl = (uint64_t *)(cand.data() + sizeof(RecHdr));
    CK(cudaMemcpyAsync(pl, c->d_best + wk * words, words * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    ch->magic = REC_MAGIC; ch->m = c->m; ch->n = c->n; ch->p = c->p; ch->ring = c->ring;
    ch->r_cap = c->R; ch->rank = (int)(key >> 54);
    ch->additions = additions_planes(c->m, c->p, pl, c->R, ch->rank);
    ch->walker_id = c->id_base + wk; ch->valid = 1;
    int32_t ff[3];
    if (ch->rank < 1 || verify_planes(c->m, c->n, c->p, c->ring, pl, c->R, ch->rank, ff) != FG_OK)
        return FG_E_INVALID_SCHEME;
    if (rec_better(ch, (const RecHdr *)c->local_rec.data())) c->local_rec.swap(cand);
    return FG_OK;
}

// local best over every walker's best scheme, from the device
int recompute_local_best(fg_ctx *c)
{
    unsigned long long key;
    int rc = device_best_key(c, &key);
    if (rc != FG_OK) return rc;
    return refresh_local_best(c, key, true);
}

}  // namespace

// host-buffer state I/O: every plane word holds at most maxlen <= 64 significant bits,
// so the current and best planes travel packed to 2, 4 or 8 bytes per word (C2: 12 of
// 48 bytes per row); a device kernel packs / unpacks around one copy each way
static int plane_width(const fg_ctx *c) { return c->maxlen <= 16 ? 2 : (c->maxlen <= 32 ? 4 : 8); }

template <class T>
__global__ void pack_planes_kernel(const uint64_t *a, const uint64_t *b, T *out, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (T)(i < n ? a[i] : b[i - n]);
}
template <class T>
__global__ void unpack_planes_kernel(const T *in, uint64_t *a, uint64_t *b, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = (uint64_t)in[i];
        if (i < n) a[i] = v; else b[i - n] = v;
    }
}

static int stage_planes(const fg_ctx *cc, bool pack)
{
    fg_ctx *c = const_cast<fg_ctx *>(cc);
    const int64_t n = (int64_t)FG_PLANES * c->R * c->W;
    const int bw = plane_width(c);
    if (!c->d_stage && cudaMalloc(&c->d_stage, (size_t)(2 * n * bw)) != cudaSuccess) {
        c->d_stage = nullptr;
        return FG_E_CUDA;
    }
    const int64_t blocks = std::min<int64_t>((2 * n + 255) / 256, (int64_t)c->num_sms * 16);
    if (bw == 2) {
        if (pack) pack_planes_kernel<uint16_t><<<(unsigned)blocks, 256, 0, c->stream>>>(c->d_cur, c->d_best, (uint16_t *)c->d_stage, n);
        else unpack_planes_kernel<uint16_t><<<(unsigned)blocks, 256, 0, c->stream>>>((const uint16_t *)c->d_stage, c->d_cur, c->d_best, n);
    } else if (bw == 4) {
        if (pack) pack_planes_kernel<uint32_t><<<(unsigned)blocks, 256, 0, c->stream>>>(c->d_cur, c->d_best, (uint32_t *)c->d_stage, n);
        else unpack_planes_kernel<uint32_t><<<(unsigned)blocks, 256, 0, c->stream>>>((const uint32_t *)c->d_stage, c->d_cur, c->d_best, n);
    } else {
        if (pack) pack_planes_kernel<uint64_t><<<(unsigned)blocks, 256, 0, c->stream>>>(c->d_cur, c->d_best, (uint64_t *)c->d_stage, n);
        else unpack_planes_kernel<uint64_t><<<(unsigned)blocks, 256, 0, c->stream>>>((const uint64_t *)c->d_stage, c->d_cur, c->d_best, n);
    }
    c->st_launches++;
    CK(cudaGetLastError());
    return FG_OK;
}

extern "C" {

void fg_params_default(fg_params *o)
{
    if (!o) return;
    o->k_flip = 16;
    o->thr_accept_eq = 42949672u;     // floor(0.01 * 2^32)
    o->thr_reduce = 2147483648u;      // 0.5
    o->thr_expand = 42949672u;        // 0.01
    o->expand_slack = 2;
    o->phase_steps = 0;
    o->flags = 0;
}

const char *fg_strerror(int s)
{
    switch (s) {
    case FG_OK: return "ok";
    case FG_E_ARG: return "bad argument";
    case FG_E_CAPACITY: return "capacity exceeded (mn|np|pm > 64, rank > r_cap or r_cap > 512)";
    case FG_E_DOMAIN: return "coefficient outside the ring, or zero factor in a seed";
    case FG_E_INVALID_SCHEME: return "scheme fails the Brent equations";
    case FG_E_CUDA: return "CUDA error";
    case FG_E_STATE: return "call out of order";
    case FG_E_UNSUPPORTED: return "no kernel for this format / r_cap in this build";
    default: return "unknown status";
    }
}

int fg_create(int m, int n, int p, int ring, int r_cap, int64_t num_walkers, int64_t walker_id_base,
              int device, void *cuda_stream, fg_ctx **out)
{
    if (!out) return FG_E_ARG;
    *out = nullptr;
    if (m < 1 || n < 1 || p < 1 || num_walkers < 1 || walker_id_base < 0 ||
        (ring != FG_ZT && ring != FG_Z2) || r_cap < 1)
        return FG_E_ARG;
    if (!format_ok(m, n, p) || r_cap > FG_MAX_RCAP) return FG_E_CAPACITY;
    if (walker_id_base + num_walkers > (1ll << 32) || num_walkers >= (1ll << 36)) return FG_E_ARG;
    const int maxlen = std::max(m * n, std::max(n * p, p * m));
    const int kind = fg_pick_kernel(ring, maxlen, r_cap);
    if (kind == FG_K_NONE) return FG_E_UNSUPPORTED;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return FG_E_CUDA;
    CK(cudaSetDevice(device));
    fg_ctx *c = new (std::nothrow) fg_ctx();
    if (!c) return FG_E_CUDA;
    c->m = m; c->n = n; c->p = p; c->ring = ring; c->R = r_cap; c->maxlen = maxlen; c->kind = kind;
    c->len[0] = m * n; c->len[1] = n * p; c->len[2] = p * m;
    c->W = num_walkers; c->id_base = walker_id_base; c->device = device;
    c->stream = (cudaStream_t)cuda_stream;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    const size_t words = (size_t)FG_PLANES * r_cap;
    // verify queue (R19): 8 entries per walker, at least 1024, at most 512 MB of entries
    // (strict improvements are rare after the first phases: C2 verifies ~900 per 10^4-step
    // phase of 16384 walkers; an overflow falls back to verifying the walker's final best
    // and is counted, fg_stats [7]; DESIGN.md section 2 "Verify-queue overflow")
    const int64_t q_budget = (int64_t)(512ll << 20) / (int64_t)(words * sizeof(uint64_t));
    c->qcap = (uint32_t)std::min<int64_t>(std::max<int64_t>(1024, std::min<int64_t>(8 * num_walkers, q_budget)), 1 << 22);
    int rc = FG_OK;
    auto alloc = [&](void **ptr, size_t bytes) {
        if (rc != FG_OK) return;
        if (cudaMalloc(ptr, bytes) != cudaSuccess) rc = FG_E_CUDA;
    };
    alloc((void **)&c->d_cur, words * num_walkers * 8);
    alloc((void **)&c->d_best, words * num_walkers * 8);
    alloc((void **)&c->d_hdr, sizeof(fg_whdr) * num_walkers);
    alloc((void **)&c->d_qplanes, words * c->qcap * 8);
    alloc((void **)&c->d_qmeta, sizeof(fg_qmeta) * c->qcap);
    alloc((void **)&c->d_misc, sizeof(DevMisc));
    alloc((void **)&c->d_task_done, sizeof(uint32_t) * (size_t)((num_walkers + 7) / 8 + 1));
    if (kind == FG_K_QL_P16 || kind == FG_K_QL_Z2)   // 5 R + R / 4 slots + 7 scalars, R <= 128
        alloc((void **)&c->d_ql_img, sizeof(uint32_t) * (size_t)(5 * 128 + 32 + 7) * num_walkers);
    if (kind == FG_K_Q4_P16 || kind == FG_K_Q4_Z2) {  // 352 slots + 8 scalars; <= 64 chunks per group
        alloc((void **)&c->d_ql_img, sizeof(uint32_t) * (size_t)(352 + 8) * num_walkers);
        alloc((void **)&c->d_ring, sizeof(uint32_t) * (size_t)((num_walkers + 7) / 8) * 64);
    }
    if (fg_kind_is_wl(kind)) alloc((void **)&c->d_wl_img, sizeof(uint32_t) * fg_wl_img_words(r_cap) * num_walkers);
    alloc((void **)&c->d_pool, words * 8);
    alloc((void **)&c->d_rank_first, sizeof(unsigned long long) * (FG_MAX_RCAP + 1));
    if (rc == FG_OK && (cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
                        cudaEventCreate(&c->ev2) != cudaSuccess))
        rc = FG_E_CUDA;
    if (rc != FG_OK) {
        cudaGetLastError();
        fg_destroy(c);
        return rc;
    }
    // unseeded walkers read as rank 0 with zero planes; the best key skips them
    if (rc == FG_OK && (cudaMemset(c->d_hdr, 0, sizeof(fg_whdr) * num_walkers) != cudaSuccess ||
                        cudaMemset(c->d_cur, 0, words * num_walkers * 8) != cudaSuccess ||
                        cudaMemset(c->d_best, 0, words * num_walkers * 8) != cudaSuccess ||
                        cudaDeviceSynchronize() != cudaSuccess))
        rc = FG_E_CUDA;
    if (rc != FG_OK) {
        cudaGetLastError();
        fg_destroy(c);
        return rc;
    }
    c->local_rec.assign(rec_bytes(r_cap), 0);
    c->pool_rec.assign(rec_bytes(r_cap), 0);
    *out = c;
    return FG_OK;
}

void fg_destroy(fg_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaFree(c->d_cur); cudaFree(c->d_best); cudaFree(c->d_hdr); cudaFree(c->d_qplanes);
    cudaFree(c->d_qmeta); cudaFree(c->d_misc); cudaFree(c->d_pool); cudaFree(c->d_task_done); cudaFree(c->d_ql_img);
    cudaFree(c->d_ring); cudaFree(c->d_stage);
    cudaFree(c->d_wl_img); cudaFree(c->d_rank_first);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->ev2) cudaEventDestroy(c->ev2);
    delete c;
}

int fg_seed_naive(fg_ctx *c)
{
    if (!c) return FG_E_ARG;
    const int rank = c->m * c->n * c->p;
    if (rank > c->R) return FG_E_CAPACITY;
    CK(cudaSetDevice(c->device));
    std::vector<uint64_t> planes((size_t)FG_PLANES * c->R, 0);
    // rows l = (i*n + j)*p + k: u = e_(i*n+j), v = e_(j*p+k), w = e_(k*m+i)
    for (int i = 0; i < c->m; ++i)
        for (int j = 0; j < c->n; ++j)
            for (int k = 0; k < c->p; ++k) {
                const int l = (i * c->n + j) * c->p + k;
                planes[0 * c->R + l] = 1ull << (i * c->n + j);
                planes[2 * c->R + l] = 1ull << (j * c->p + k);
                planes[4 * c->R + l] = 1ull << (k * c->m + i);
            }
    return seed_planes(c, planes.data(), rank, 0, c->W);
}

int fg_seed_pool(fg_ctx *c, const int8_t *coeffs, int rank, int64_t w0, int64_t w1)
{
    if (!c || !coeffs || w0 < 0 || w1 > c->W || w0 >= w1) return FG_E_ARG;
    if (rank < 1 || rank > c->R) return FG_E_CAPACITY;
    std::vector<uint64_t> planes((size_t)FG_PLANES * c->R, 0);
    int rc = pack_planes(c->m, c->n, c->p, c->ring, coeffs, rank, c->R, planes.data());
    if (rc != FG_OK) return rc;
    if (has_zero_factor(planes.data(), c->R, rank)) return FG_E_DOMAIN;
    int32_t ff[3];
    rc = verify_planes(c->m, c->n, c->p, c->ring, planes.data(), c->R, rank, ff);
    if (rc != FG_OK) return rc;
    if (c->ring == FG_ZT) normalize_planes(planes.data(), c->R, rank);
    CK(cudaSetDevice(c->device));
    return seed_planes(c, planes.data(), rank, w0, w1);
}

int fg_load_walkers(fg_ctx *c, const int8_t *coeffs, const int32_t *ranks, int64_t w_begin, int64_t count)
{
    if (!c || !coeffs || !ranks || w_begin < 0 || count < 1 || w_begin + count > c->W) return FG_E_ARG;
    const size_t words = (size_t)FG_PLANES * c->R;
    const int w = width_of(c->m, c->n, c->p);
    std::vector<uint64_t> planes(words * count);
    std::vector<fg_whdr> hdr(count);
    for (int64_t k = 0; k < count; ++k) {
        const int rank = ranks[k];
        if (rank < 1 || rank > c->R) return FG_E_CAPACITY;
        uint64_t *pl = planes.data() + k * words;
        int rc = pack_planes(c->m, c->n, c->p, c->ring, coeffs + (size_t)k * c->R * w, rank, c->R, pl);
        if (rc != FG_OK) return rc;
        if (has_zero_factor(pl, c->R, rank)) return FG_E_DOMAIN;
        int32_t ff[3];
        rc = verify_planes(c->m, c->n, c->p, c->ring, pl, c->R, rank, ff);
        if (rc != FG_OK) return rc;
        if (c->ring == FG_ZT) normalize_planes(pl, c->R, rank);
        memset(&hdr[k], 0, sizeof(fg_whdr));
        hdr[k].r = rank;
        hdr[k].best_r = rank;
        hdr[k].digest = 0xcbf29ce484222325ULL;
        hdr[k].best_adds = additions_planes(c->m, c->p, pl, c->R, rank);
    }
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpyAsync(c->d_cur + w_begin * words, planes.data(), words * count * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_best + w_begin * words, planes.data(), words * count * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_hdr + w_begin, hdr.data(), sizeof(fg_whdr) * count, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    mark_covered(c, w_begin, w_begin + count);
    c->img_valid = false;
    if (c->seeded) {
        int rmin = FG_MAX_RCAP;
        for (int64_t k = 0; k < count; ++k) rmin = std::min(rmin, (int)ranks[k]);
        int rr = reset_rank_first(c, rmin);
        if (rr != FG_OK) return rr;
    }
    if (!c->seeded) return FG_OK;
    return recompute_local_best(c);
}

int fg_walk(fg_ctx *c, uint64_t steps, uint64_t seed, const fg_params *prm)
{
    if (!c) return FG_E_ARG;
    if (!c->seeded) return FG_E_STATE;
    fg_params P;
    if (prm) P = *prm; else fg_params_default(&P);
    if (P.k_flip < 1 || P.k_flip > FG_MAX_KFLIP || (P.flags & ~FG_FLAG_COMPLEXITY) || P.expand_slack < -FG_MAX_RCAP)
        return FG_E_ARG;
    CK(cudaSetDevice(c->device));
    WalkArgs a;
    memset(&a, 0, sizeof(a));
    a.cur = c->d_cur; a.best = c->d_best; a.hdr = c->d_hdr;
    a.num_walkers = c->W; a.id_base = c->id_base;
    a.m = c->m; a.n = c->n; a.p = c->p; a.R = c->R;
    a.len_u = c->len[0]; a.len_v = c->len[1]; a.len_w = c->len[2]; a.mp = c->m * c->p;
    a.seed = seed;
    a.mode = (P.flags & FG_FLAG_COMPLEXITY) ? 1u : 0u;
    a.k_flip = P.k_flip; a.thr_eq = P.thr_accept_eq; a.thr_reduce = P.thr_reduce;
    a.thr_expand = P.thr_expand; a.slack = P.expand_slack;
    a.q_planes = c->d_qplanes; a.q_meta = c->d_qmeta; a.q_count = &c->d_misc->q_count;
    a.q_cap = c->qcap; a.q_overflow = &c->d_misc->q_overflow; a.best_key = &c->d_misc->best_key;
    a.work_counter = &c->d_misc->work_counter;
    a.task_done = c->d_task_done;
    a.ql_img = c->d_ql_img;
    a.ring = c->d_ring;
    a.ring_tail = &c->d_misc->ring_tail;
    a.wl_img = c->d_wl_img;
    // the complexity mode (R24): walk_wl / walk_wm pick their CM instance from a.mode,
    // walk_ql contexts run it on walk_wl, walk_q4 / walk_w32 on their CM instance
    int kind = c->kind;
    if (a.mode && !fg_kind_is_wl(kind)) kind = fg_kind_for_mode(kind);
    a.dbg = getenv("FG_DBG") ? (uint32_t)strtoul(getenv("FG_DBG"), nullptr, 0) : 0u;
    a.dbgbuf = c->d_misc->dbgbuf;
    VerifyArgs v;
    memset(&v, 0, sizeof(v));
    v.planes = c->d_qplanes; v.meta = c->d_qmeta; v.count_ptr = &c->d_misc->q_count; v.cap = c->qcap;
    v.m = c->m; v.n = c->n; v.p = c->p; v.R = c->R; v.ring = c->ring; v.hdr = c->d_hdr;
    v.fail_count = &c->d_misc->verify_fail;

    CK(cudaMemsetAsync(c->d_misc, 0, sizeof(DevMisc), c->stream));
    uint64_t remaining = steps;
    uint64_t verified = 0;
    float walk_ms = 0.f, ver_ms = 0.f;
    DevMisc hm;
    do {
        const uint64_t chunk = (P.phase_steps && remaining > P.phase_steps) ? P.phase_steps : remaining;
        a.steps = chunk;
        CK(cudaMemsetAsync(&c->d_misc->best_key, 0xff, sizeof(unsigned long long), c->stream));
        CK(cudaMemsetAsync(&c->d_misc->q_count, 0, sizeof(uint32_t), c->stream));
        CK(cudaMemsetAsync(&c->d_misc->work_counter, 0, 2 * sizeof(unsigned long long), c->stream));
        CK(cudaMemsetAsync(c->d_task_done, 0, sizeof(uint32_t) * (size_t)((c->W + 7) / 8 + 1), c->stream));
        CK(cudaEventRecord(c->ev0, c->stream));
        a.img_valid = c->img_valid ? 1u : 0u;
        CK(fg_launch_walk(kind, a, c->num_sms, c->stream));
        c->img_valid = fg_kind_is_wl(kind) && a.wl_img != nullptr;   // R24 on walk_ql contexts: no image
        CK(cudaEventRecord(c->ev1, c->stream));
        CK(fg_launch_verify(v, c->stream));
        CK(cudaEventRecord(c->ev2, c->stream));
        if (a.mode == 0) {
            CK(fg_launch_rank_first(c->d_qmeta, &c->d_misc->q_count, c->qcap, c->d_rank_first, c->stream));
            c->st_launches++;
        }
        c->st_launches += 2;
        c->st_walk_launches++;
        CK(cudaMemcpyAsync(&hm, c->d_misc, sizeof(hm), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        float t1 = 0.f, t2 = 0.f;
        cudaEventElapsedTime(&t1, c->ev0, c->ev1);
        cudaEventElapsedTime(&t2, c->ev1, c->ev2);
        walk_ms += t1;
        ver_ms += t2;
        verified += std::min(hm.q_count, c->qcap);
        remaining -= chunk;
    } while (remaining > 0);
    if (a.dbg && hm.dbgbuf[0]) {
        // FG_DBG structure self-check failed: report and fail the call
        fprintf(stderr, "libfg dbg: %u %u %u %u %u %u %u %u %u %u\n", hm.dbgbuf[0], hm.dbgbuf[1], hm.dbgbuf[2],
                hm.dbgbuf[3], hm.dbgbuf[4], hm.dbgbuf[5], hm.dbgbuf[6], hm.dbgbuf[7], hm.dbgbuf[8], hm.dbgbuf[9]);
        return FG_E_STATE;
    }
    if (hm.q_overflow) {
        // strict improvements that missed the queue: verify those walkers' final bests
        CK(cudaMemsetAsync(&c->d_misc->restarted, 0, sizeof(unsigned long long), c->stream));
        CK(fg_launch_verify_flagged(c->d_best, c->d_hdr, c->W, c->R, c->m, c->n, c->p, c->ring,
                                    &c->d_misc->verify_fail, &c->d_misc->restarted, c->stream));
        c->st_launches++;
        CK(cudaMemcpyAsync(&hm, c->d_misc, sizeof(hm), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        verified += hm.restarted;
    }
    // a walker whose strict improvement failed the Brent check never supplies the
    // local best (R19): the key is recomputed without the failing walkers
    unsigned long long key = hm.best_key;
    if (hm.verify_fail) {
        int rk = device_best_key(c, &key);
        if (rk != FG_OK) return rk;
    }
    int rc = refresh_local_best(c, key, false);
    c->st_vfail += hm.verify_fail;
    c->st_overflow += hm.q_overflow;
    c->st_steps += steps * (uint64_t)c->W;
    c->st_verified += verified;
    c->st_walk_us += (uint64_t)(walk_ms * 1000.0);
    c->st_verify_us += (uint64_t)(ver_ms * 1000.0);
    return rc;
}

int fg_verify(int m, int n, int p, int ring, const int8_t *coeffs, int rank, int32_t first_fail[3])
{
    if (first_fail) first_fail[0] = first_fail[1] = first_fail[2] = -1;
    if (m < 1 || n < 1 || p < 1 || rank < 0 || (rank > 0 && !coeffs) || (ring != FG_ZT && ring != FG_Z2))
        return FG_E_ARG;
    if (!format_ok(m, n, p)) return FG_E_CAPACITY;
    const int R = std::max(rank, 1);
    std::vector<uint64_t> planes((size_t)FG_PLANES * R, 0);
    int rc = pack_planes(m, n, p, ring, coeffs, rank, R, planes.data());
    if (rc != FG_OK) return rc;
    return verify_planes(m, n, p, ring, planes.data(), R, rank, first_fail);
}

int fg_verify_batch(fg_ctx *c, const int8_t *coeffs, const int32_t *ranks, int64_t count,
                    int32_t *ok_out, int32_t *ff_out)
{
    if (!c || !coeffs || !ranks || count < 0 || !ok_out) return FG_E_ARG;
    if (count == 0) return FG_OK;
    const int R = c->R, w = width_of(c->m, c->n, c->p);
    const size_t words = (size_t)FG_PLANES * R;
    std::vector<uint64_t> planes(words * count);
    std::vector<fg_qmeta> meta(count);
    for (int64_t k = 0; k < count; ++k) {
        if (ranks[k] < 0 || ranks[k] > R) return FG_E_CAPACITY;
        int rc = pack_planes(c->m, c->n, c->p, c->ring, coeffs + (size_t)k * R * w, ranks[k], R,
                             planes.data() + k * words);
        if (rc != FG_OK) return rc;
        memset(&meta[k], 0, sizeof(fg_qmeta));
        meta[k].rank = ranks[k];
        meta[k].walker = k;
    }
    CK(cudaSetDevice(c->device));
    uint64_t *dp = nullptr;
    fg_qmeta *dm = nullptr;
    CK(cudaMallocAsync((void **)&dp, words * count * 8, c->stream));
    CK(cudaMallocAsync((void **)&dm, sizeof(fg_qmeta) * count, c->stream));
    CK(cudaMemcpyAsync(dp, planes.data(), words * count * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dm, meta.data(), sizeof(fg_qmeta) * count, cudaMemcpyHostToDevice, c->stream));
    VerifyArgs v;
    memset(&v, 0, sizeof(v));
    v.planes = dp; v.meta = dm; v.count_ptr = nullptr; v.count = (uint32_t)count; v.cap = (uint32_t)count;
    v.m = c->m; v.n = c->n; v.p = c->p; v.R = R; v.ring = c->ring;
    CK(fg_launch_verify(v, c->stream));
    c->st_launches++;
    CK(cudaMemcpyAsync(meta.data(), dm, sizeof(fg_qmeta) * count, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaFreeAsync(dp, c->stream));
    CK(cudaFreeAsync(dm, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t k = 0; k < count; ++k) {
        ok_out[k] = meta[k].ok;
        if (ff_out) for (int t = 0; t < 3; ++t) ff_out[3 * k + t] = meta[k].ff[t];
    }
    return FG_OK;
}

int fg_best(const fg_ctx *c, int *rank, int *adds, int64_t *walker_id, int8_t *coeffs_out)
{
    if (!c) return FG_E_ARG;
    const RecHdr *l = (const RecHdr *)c->local_rec.data();
    const RecHdr *pl = (const RecHdr *)c->pool_rec.data();
    const RecHdr *b = rec_better(pl, l) ? pl : l;
    if (!b->valid) return FG_E_STATE;
    if (rank) *rank = b->rank;
    if (adds) *adds = b->additions;
    if (walker_id) *walker_id = b->walker_id;
    if (coeffs_out) {
        memset(coeffs_out, 0, (size_t)c->R * width_of(c->m, c->n, c->p));
        unpack_planes(c->m, c->n, c->p, (const uint64_t *)(b + 1), c->R, b->rank, coeffs_out);
    }
    return FG_OK;
}

int fg_get_walkers(const fg_ctx *c, int64_t w0, int64_t w1, int32_t *r, int32_t *best_r, int32_t *best_adds,
                   uint64_t *digest, uint64_t *step, uint64_t *cnt, int8_t *rows, int8_t *best)
{
    if (!c || w0 < 0 || w1 > c->W || w0 > w1) return FG_E_ARG;
    if (w0 == w1) return FG_OK;
    const int64_t nw = w1 - w0;
    const size_t words = (size_t)FG_PLANES * c->R;
    const int w = width_of(c->m, c->n, c->p);
    CK(cudaSetDevice(c->device));
    std::vector<fg_whdr> h(nw);
    CK(cudaMemcpyAsync(h.data(), c->d_hdr + w0, sizeof(fg_whdr) * nw, cudaMemcpyDeviceToHost, c->stream));
    std::vector<uint64_t> pc, pb;
    if (rows) {
        pc.resize(words * nw);
        CK(cudaMemcpyAsync(pc.data(), c->d_cur + w0 * words, words * nw * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    if (best) {
        pb.resize(words * nw);
        CK(cudaMemcpyAsync(pb.data(), c->d_best + w0 * words, words * nw * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t k = 0; k < nw; ++k) {
        if (r) r[k] = h[k].r;
        if (best_r) best_r[k] = h[k].best_r;
        if (best_adds) best_adds[k] = h[k].best_adds;
        if (digest) digest[k] = h[k].digest;
        if (step) step[k] = h[k].step;
        if (cnt) memcpy(cnt + k * FG_NCNT, h[k].cnt, sizeof(uint64_t) * FG_NCNT);
        if (rows) {
            int8_t *dst = rows + (size_t)k * c->R * w;
            memset(dst, 0, (size_t)c->R * w);
            unpack_planes(c->m, c->n, c->p, pc.data() + k * words, c->R, h[k].r, dst);
        }
        if (best) {
            int8_t *dst = best + (size_t)k * c->R * w;
            memset(dst, 0, (size_t)c->R * w);
            unpack_planes(c->m, c->n, c->p, pb.data() + k * words, c->R, h[k].best_r, dst);
        }
    }
    return FG_OK;
}

int fg_get_walker(const fg_ctx *c, int64_t wk, int *rank, int *best_rank, uint64_t *digest,
                  int8_t *coeffs_out, int8_t *best_out)
{
    int32_t r = 0, br = 0;
    int rc = fg_get_walkers(c, wk, wk + 1, &r, &br, nullptr, digest, nullptr, nullptr, coeffs_out, best_out);
    if (rc != FG_OK) return rc;
    if (rank) *rank = r;
    if (best_rank) *best_rank = br;
    return FG_OK;
}

size_t fg_record_bytes(int r_cap) { return (r_cap < 1 || r_cap > FG_MAX_RCAP) ? 0 : rec_bytes(r_cap); }

int fg_export_best(const fg_ctx *c, void *record)
{
    if (!c || !record) return FG_E_ARG;
    const RecHdr *l = (const RecHdr *)c->local_rec.data();
    if (!l->valid) return FG_E_STATE;
    memcpy(record, c->local_rec.data(), c->local_rec.size());
    return FG_OK;
}

int fg_record_merge(const void *records, int count, void *out)
{
    if (!records || !out || count < 1) return FG_E_ARG;
    const RecHdr *h0 = (const RecHdr *)records;
    if (h0->magic != REC_MAGIC || h0->r_cap < 1 || h0->r_cap > FG_MAX_RCAP) return FG_E_ARG;
    const size_t sz = rec_bytes(h0->r_cap);
    const unsigned char *base = (const unsigned char *)records;
    int bestk = -1;
    for (int k = 0; k < count; ++k) {
        const RecHdr *h = (const RecHdr *)(base + k * sz);
        if (h->magic != REC_MAGIC || h->r_cap != h0->r_cap || h->m != h0->m || h->n != h0->n ||
            h->p != h0->p || h->ring != h0->ring)
            return FG_E_ARG;
        if (!h->valid) continue;
        if (bestk < 0 || rec_better(h, (const RecHdr *)(base + bestk * sz))) bestk = k;
    }
    if (bestk < 0) {
        memcpy(out, base, sz);
        ((RecHdr *)out)->valid = 0;
        return FG_OK;
    }
    memcpy(out, base + bestk * sz, sz);
    return FG_OK;
}

int fg_import_best(fg_ctx *c, const void *records, int count)
{
    if (!c || !records || count < 1) return FG_E_ARG;
    const RecHdr *h0 = (const RecHdr *)records;
    if (h0->magic != REC_MAGIC || h0->r_cap != c->R || h0->m != c->m || h0->n != c->n || h0->p != c->p ||
        h0->ring != c->ring)
        return FG_E_ARG;
    std::vector<unsigned char> merged(rec_bytes(c->R));
    int rc = fg_record_merge(records, count, merged.data());
    if (rc != FG_OK) return rc;
    const RecHdr *mh = (const RecHdr *)merged.data();
    if (!mh->valid) return FG_OK;
    // imported schemes are checked before they enter the pool (R19)
    int32_t ff[3];
    if (verify_planes(c->m, c->n, c->p, c->ring, (const uint64_t *)(mh + 1), c->R, mh->rank, ff) != FG_OK)
        return FG_E_INVALID_SCHEME;
    if (rec_better(mh, (const RecHdr *)c->pool_rec.data())) c->pool_rec = merged;
    return FG_OK;
}

int fg_record_pack(int m, int n, int p, int ring, int r_cap, const int8_t *coeffs, int rank, int64_t walker_id,
                   void *record)
{
    if (!record || !coeffs || r_cap < 1 || r_cap > FG_MAX_RCAP || rank < 1 || rank > r_cap) return FG_E_ARG;
    if (!format_ok(m, n, p)) return FG_E_CAPACITY;
    RecHdr *h = (RecHdr *)record;
    memset(h, 0, sizeof(*h));
    uint64_t *pl = (uint64_t *)(h + 1);
    int rc = pack_planes(m, n, p, ring, coeffs, rank, r_cap, pl);
    if (rc != FG_OK) return rc;
    h->magic = REC_MAGIC; h->m = m; h->n = n; h->p = p; h->ring = ring; h->r_cap = r_cap;
    h->rank = rank; h->additions = additions_planes(m, p, pl, r_cap, rank); h->walker_id = walker_id;
    h->valid = 1;
    return FG_OK;
}

int fg_record_unpack(const void *record, int *m, int *n, int *p, int *ring, int *rank, int *additions,
                     int64_t *walker_id, int8_t *coeffs_out)
{
    if (!record) return FG_E_ARG;
    const RecHdr *h = (const RecHdr *)record;
    if (h->magic != REC_MAGIC) return FG_E_ARG;
    if (m) *m = h->m;
    if (n) *n = h->n;
    if (p) *p = h->p;
    if (ring) *ring = h->ring;
    if (rank) *rank = h->valid ? h->rank : 0;
    if (additions) *additions = h->additions;
    if (walker_id) *walker_id = h->walker_id;
    if (coeffs_out && h->valid)
        unpack_planes(h->m, h->n, h->p, (const uint64_t *)(h + 1), h->r_cap, h->rank, coeffs_out);
    return FG_OK;
}

int fg_restart(fg_ctx *c, int slack, int64_t *restarted)
{
    if (!c || slack < 0) return FG_E_ARG;
    if (!c->seeded) return FG_E_STATE;
    const RecHdr *pl = (const RecHdr *)c->pool_rec.data();
    const RecHdr *l = (const RecHdr *)c->local_rec.data();
    const RecHdr *b = rec_better(pl, l) ? pl : l;
    if (restarted) *restarted = 0;
    if (!b->valid) return FG_OK;
    CK(cudaSetDevice(c->device));
    const size_t words = (size_t)FG_PLANES * c->R;
    CK(cudaMemcpyAsync(c->d_pool, (const uint64_t *)(b + 1), words * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(&c->d_misc->restarted, 0, sizeof(unsigned long long), c->stream));
    CK(fg_launch_restart(c->d_cur, c->d_best, c->d_hdr, c->W, c->R, c->d_pool, b->rank, b->additions, slack,
                         &c->d_misc->restarted, c->stream));
    c->img_valid = false;
    c->st_launches++;
    unsigned long long n = 0;
    CK(cudaMemcpyAsync(&n, &c->d_misc->restarted, sizeof(n), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (restarted) *restarted = (int64_t)n;
    return recompute_local_best(c);
}

// walk_wl's class image travels with the state (a checkpoint resumes without rebuilding
// the class lists); other kernels have none
static size_t img_bytes(const fg_ctx *c)
{
    return c->d_wl_img ? fg_wl_img_words(c->R) * 4 * (size_t)c->W : 0;
}

size_t fg_state_bytes(const fg_ctx *c)
{
    if (!c) return 0;
    const size_t words = (size_t)FG_PLANES * c->R;
    return 64 + sizeof(fg_whdr) * c->W + 2 * words * plane_width(c) * c->W + img_bytes(c);
}

int fg_save_state(const fg_ctx *c, void *buf)
{
    if (!c || !buf) return FG_E_ARG;
    if (!c->seeded) return FG_E_STATE;
    CK(cudaSetDevice(c->device));
    const size_t words = (size_t)FG_PLANES * c->R;
    const size_t pb = 2 * words * plane_width(c) * c->W;
    unsigned char *b = (unsigned char *)buf;
    const size_t ib = img_bytes(c);
    uint32_t hdr[16] = {STATE_MAGIC, (uint32_t)c->m, (uint32_t)c->n, (uint32_t)c->p, (uint32_t)c->ring,
                        (uint32_t)c->R, (uint32_t)(c->W & 0xffffffff), (uint32_t)(c->W >> 32),
                        (uint32_t)(ib ? fg_wl_img_words(c->R) : 0), (uint32_t)(ib && c->img_valid),
                        (uint32_t)plane_width(c)};
    memcpy(b, hdr, 64);
    const int rc = stage_planes(c, true);
    if (rc != FG_OK) return rc;
    CK(cudaMemcpyAsync(b + 64, c->d_hdr, sizeof(fg_whdr) * c->W, cudaMemcpyDeviceToHost, c->stream));
    unsigned char *pc = b + 64 + sizeof(fg_whdr) * c->W;
    CK(cudaMemcpyAsync(pc, c->d_stage, pb, cudaMemcpyDeviceToHost, c->stream));
    if (ib) CK(cudaMemcpyAsync(pc + pb, c->d_wl_img, ib, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FG_OK;
}

int fg_load_state(fg_ctx *c, const void *buf)
{
    if (!c || !buf) return FG_E_ARG;
    const uint32_t *hdr = (const uint32_t *)buf;
    if (hdr[0] != STATE_MAGIC || (int)hdr[1] != c->m || (int)hdr[2] != c->n || (int)hdr[3] != c->p ||
        (int)hdr[4] != c->ring || (int)hdr[5] != c->R ||
        ((int64_t)hdr[6] | ((int64_t)hdr[7] << 32)) != c->W || (int)hdr[10] != plane_width(c))
        return FG_E_ARG;
    CK(cudaSetDevice(c->device));
    const size_t words = (size_t)FG_PLANES * c->R;
    const size_t pb = 2 * words * plane_width(c) * c->W;
    const unsigned char *b = (const unsigned char *)buf;
    if (!c->d_stage && cudaMalloc(&c->d_stage, pb) != cudaSuccess) {
        c->d_stage = nullptr;
        return FG_E_CUDA;
    }
    CK(cudaMemcpyAsync(c->d_hdr, b + 64, sizeof(fg_whdr) * c->W, cudaMemcpyHostToDevice, c->stream));
    const unsigned char *pc = b + 64 + sizeof(fg_whdr) * c->W;
    CK(cudaMemcpyAsync(c->d_stage, pc, pb, cudaMemcpyHostToDevice, c->stream));
    const int rc = stage_planes(c, false);
    if (rc != FG_OK) return rc;
    // a class image saved by the same kind of context resumes as it was saved
    const size_t ib = img_bytes(c);
    const bool img = ib && hdr[8] == (uint32_t)fg_wl_img_words(c->R) && hdr[9] == 1u;
    if (img) CK(cudaMemcpyAsync(c->d_wl_img, pc + pb, ib, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->covered.assign(1, {0, c->W});
    c->img_valid = img;
    c->seeded = true;
    return recompute_local_best(c);
}

int fg_stats(const fg_ctx *c, uint64_t out[12])
{
    if (!c || !out) return FG_E_ARG;
    uint64_t tot[FG_NCNT] = {0};
    if (c->seeded) {
        CK(cudaSetDevice(c->device));
        std::vector<fg_whdr> h(c->W);
        CK(cudaMemcpyAsync(h.data(), c->d_hdr, sizeof(fg_whdr) * c->W, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (const fg_whdr &x : h)
            for (int k = 0; k < FG_NCNT; ++k) tot[k] += x.cnt[k];
    }
    out[0] = tot[FG_CNT_STEPS];
    out[1] = tot[FG_CNT_DRAWS];
    out[2] = tot[FG_CNT_FLIPS];
    out[3] = tot[FG_CNT_EXPAND_OK];
    out[4] = tot[FG_CNT_MERGES] + tot[FG_CNT_ZERO_REMOVED];
    out[5] = c->st_verified;
    out[6] = c->st_vfail;
    out[7] = c->st_overflow;
    out[8] = c->st_launches;
    out[9] = c->st_walk_us;
    out[10] = c->st_verify_us;
    out[11] = c->st_walk_launches;
    return FG_OK;
}

int fg_rank_first_steps(const fg_ctx *c, int max_rank, uint64_t *out)
{
    if (!c || !out || max_rank < 0) return FG_E_ARG;
    if (!c->seeded) return FG_E_STATE;
    CK(cudaSetDevice(c->device));
    std::vector<unsigned long long> v(FG_MAX_RCAP + 1);
    CK(cudaMemcpyAsync(v.data(), c->d_rank_first, v.size() * sizeof(v[0]), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k <= max_rank; ++k) out[k] = k <= FG_MAX_RCAP ? (uint64_t)v[k] : ~0ull;
    return FG_OK;
}

const char *fg_kernel_name(const fg_ctx *c) { return c ? fg_kernel_kind_name(c->kind) : "none"; }

}  // extern "C"
