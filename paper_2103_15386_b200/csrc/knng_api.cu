// knng_api.cu -- the C ABI of include/knng.h: validation, workspace layout,
// stream-ordered orchestration of the kernels, error mapping, counters.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <functional>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/knng.h"
#include "comm.cuh"
#include "dist_kernels.cuh"
#include "eval_kernels.cuh"
#include "ggm_kernels.cuh"
#include "join_kernel.cuh"
#include "join_tc.cuh"
#include "join_tcf.cuh"
#include "join_locked.cuh"
#include "seg_kernels.cuh"
#include "join_ws.cuh"

using namespace knng;

namespace {

thread_local std::string g_err;
thread_local std::vector<knng_iter_stats> g_last_stats;
std::atomic<int64_t> g_launches{0};
std::atomic<int> g_timing{0};
std::atomic<int> g_opt_exact_u8{1};
std::atomic<int> g_opt_join_kernel{0};
std::atomic<int> g_opt_update{0};  // 0 bulk (default), 1 full (GNND-r1), 2 locked, 3 locked, one lock per list
thread_local int g_last_exact_u8 = 0;
std::mutex g_time_mu;
std::map<std::string, std::pair<double, int64_t>> g_times;

knng_status fail(knng_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

constexpr int kMaxIters = 256;
#ifndef KNNG_FUSED_INIT
#define KNNG_FUSED_INIT 1
#endif
#ifndef KNNG_FUSED_U8
#define KNNG_FUSED_U8 1
#endif
#ifndef KNNG_REV_SCATTER4
#define KNNG_REV_SCATTER4 1
#endif
constexpr bool g_rev_scatter4 = KNNG_REV_SCATTER4 != 0;

// ---------------------------------------------------------------- layout
struct Layout {
    size_t keys, newmask, kth, lock, imask, bcnt, bucket, fwd, fcnt, rcnt, fpos, off, rsrc, G, gcnt, bsum, cand, stats,
        xnorm, xu8, sqn, reserved, flag, total;
    bool has_cand;
};

int64_t scan_blocks(int64_t n) { return (n + kScanBlock - 1) / kScanBlock; }

size_t align_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

Layout make_layout(int64_t n, int d, int k, int p, bool xcopy, bool own_keys, bool merge, bool u8copy = false) {
    Layout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t at = off;
        off += align_up(bytes);
        return at;
    };
    const int cap = 2 * p;
    L.keys = own_keys ? take(static_cast<size_t>(n) * k * 8) : 0;
    L.newmask = take(static_cast<size_t>(n) * (k > 32 ? k / 32 : 1) * 4);
    L.kth = take(static_cast<size_t>(n) * 8);
    const int segs = k > 32 ? k / 32 : 1;                    // list segments (D40)
    L.lock = take(static_cast<size_t>(n) * segs * 4);        // locked update (option "update")
    L.imask = take(static_cast<size_t>(n) * segs * 4);
    L.bcnt = take(static_cast<size_t>(n) * 4);
    // bucket capacity: sum_t [2 (|R_new(t)| + |F_new(t)|) + |R_old(t)| + |F_old(t)|] <= 6 n p
    L.bucket = take(static_cast<size_t>(6) * n * p * 8);
    L.fwd = take(static_cast<size_t>(2) * n * p * 4);
    L.fcnt = take(static_cast<size_t>(n) * 2);
    L.rcnt = take(static_cast<size_t>(2) * n * 4);
    L.fpos = take(static_cast<size_t>(2) * n * p * 4);
    L.off = take(static_cast<size_t>(3) * (n + 1) * 8);
    L.rsrc = take(static_cast<size_t>(2) * n * p * 4);
    L.G = take(static_cast<size_t>(2) * n * cap * 4);
    L.gcnt = take(static_cast<size_t>(n) * 2);
    L.bsum = take(static_cast<size_t>(3) * scan_blocks(n) * 8);
    // join output staging: only the legacy batched join (option join_kernel 1,
    // or rows that are not whole 16-B chunks) files through it; the other joins
    // file inside the kernel.  (A misaligned base pointer allocates it lazily.)
    L.has_cand = g_opt_join_kernel.load() == 1 || d % 16 != 0;
    L.cand = L.has_cand ? take(static_cast<size_t>(n) * 3 * cap * 8) : 0;
    L.stats = take(sizeof(DevStats) * kMaxIters);
    L.xnorm = xcopy ? take(static_cast<size_t>(n) * d * 4) : 0;  // normalised (cosine) / float (chi2 of u8) rows
    L.reserved = merge ? take(static_cast<size_t>(n) * (k / 2 > 0 ? k / 2 : 1) * 8) : 0;
    L.xu8 = u8copy ? take(static_cast<size_t>(n) * d) : 0;  // exact integer copy (option exact_u8)
    L.sqn = take(static_cast<size_t>(n) * 4);                // exact squared norms (uint8 tensor-core join)
    L.flag = take(16);
    L.total = off;
    return L;
}

// 2-D TMA descriptor of uint8 rows [n][d] (d % 16 == 0, d <= 128): box of
// one 128-B row, SW128 swizzle (the tensor-core join's shared-memory layout;
// columns past d are zero-filled as out of bounds).  false if the driver
// entry point is unavailable.
PFN_cuTensorMapEncodeTiled tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        cudaGetLastError();
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }();
    return encode;
}
bool make_row_tmap(const void* X, int64_t n, int d, CUtensorMap* tm) {
    PFN_cuTensorMapEncodeTiled encode = tmap_encoder();
    if (!encode) return false;
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(d)};
    const cuuint32_t box[2] = {128, 1};
    const cuuint32_t estride[2] = {1, 1};
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(X), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D TMA descriptor of float rows [n][d] (d % 4 == 0): box of one 128-B
// slab (32 floats) of one row, SW128 swizzle (the float join's ring layout);
// columns past d are zero-filled as out of bounds.
[[maybe_unused]] bool make_f32_slab_tmap(const float* X, int64_t n, int d, CUtensorMap* tm) {
    PFN_cuTensorMapEncodeTiled encode = tmap_encoder();
    if (!encode) return false;
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(d) * 4};
    const cuuint32_t box[2] = {32, 1};
    const cuuint32_t estride[2] = {1, 1};
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- context
struct Ctx {
    cudaStream_t stream = nullptr;
    bool timing = false;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    void* owned_ws = nullptr;
    void* owned_extra = nullptr;  // lazily allocated join staging (misaligned rows)
    cudaError_t err = cudaSuccess;
    std::string err_where;

    cudaEvent_t ev() {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        pool.push_back(e);
        return e;
    }
    ~Ctx() {
        for (auto e : pool) cudaEventDestroy(e);
        if (owned_ws) cudaFreeAsync(owned_ws, stream);
        if (owned_extra) cudaFreeAsync(owned_extra, stream);
    }
    // launch bookkeeping: count, optional events, error capture
    template <typename F>
    bool launch(const char* name, F&& f) {
        if (err != cudaSuccess) return false;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timing) {
            e0 = ev();
            if (e0) cudaEventRecord(e0, stream);
        }
        f();
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (timing) {
            e1 = ev();
            if (e1) cudaEventRecord(e1, stream);
            if (e0 && e1) marks.push_back({name, {e0, e1}});
        }
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            err = e;
            err_where = name;
            return false;
        }
        return true;
    }
    knng_status finish() {
        const cudaError_t se = cudaStreamSynchronize(stream);
        if (err == cudaSuccess && se != cudaSuccess) {
            err = se;
            err_where = "stream synchronize";
        }
        if (err != cudaSuccess)
            return fail(KNNG_E_CUDA, "CUDA error in %s: %s", err_where.c_str(), cudaGetErrorString(err));
        if (timing) {
            std::lock_guard<std::mutex> lk(g_time_mu);
            for (auto& m : marks) {
                float ms = 0.f;
                if (cudaEventElapsedTime(&ms, m.second.first, m.second.second) == cudaSuccess) {
                    auto& t = g_times[m.first];
                    t.first += ms;
                    t.second += 1;
                }
            }
        }
        return KNNG_OK;
    }
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// rows copied into L.xnorm: normalised rows (cosine, D6), float rows of uint8
// input (chi-square is evaluated in float, D39)
bool needs_xcopy(knng_metric metric, knng_dtype dt) {
    return metric == KNNG_COSINE || (metric == KNNG_CHI2 && dt == KNNG_U8);
}

knng_status check_common(knng_dtype dt, int64_t n, int32_t d, int32_t k, knng_metric metric, int32_t p) {
    if (dt != KNNG_F32 && dt != KNNG_U8) return fail(KNNG_E_USAGE, "unknown dtype %d", static_cast<int>(dt));
    if (metric != KNNG_L2SQ && metric != KNNG_COSINE && metric != KNNG_CHI2)
        return fail(KNNG_E_USAGE, "unknown metric %d", static_cast<int>(metric));
    if (metric == KNNG_COSINE && dt != KNNG_F32) return fail(KNNG_E_USAGE, "cosine requires float32 vectors");
    if (d < 1) return fail(KNNG_E_USAGE, "d must be >= 1 (got %d)", d);
    if (k < 2 || (k > 32 && (k % 32 != 0 || k > 128)))
        return fail(KNNG_E_USAGE, "k must be in [2, 32] or 64, 96, 128 (segmented lists, P:246) (got %d)", k);
    if (p < 1 || p >= k) return fail(KNNG_E_USAGE, "sample_size must satisfy 1 <= p < k (got p=%d, k=%d)", p, k);
    if (2 * p > 32) return fail(KNNG_E_USAGE, "sample_size must be <= 16 in this version (got %d)", p);
    if (n <= k) return fail(KNNG_E_USAGE, "n must exceed k (n=%lld, k=%d)", static_cast<long long>(n), k);
    if (k > 32 && n < k + k / 32)
        return fail(KNNG_E_USAGE, "segmented lists need n >= k + k/32 (each residue class holds 32 others)");
    if (n >= 0xFFFFFFFFll) return fail(KNNG_E_USAGE, "n must be < 2^32 - 1");
    if (n * static_cast<int64_t>(p) >= (1ll << 32)) return fail(KNNG_E_USAGE, "n * sample_size must be < 2^32");
    return KNNG_OK;
}

struct Run {
    Ctx& c;
    Layout L;
    char* ws;
    Dims D;
    Graph G;
    Samples S;
    DevStats* stats;
    const void* X;
    knng_dtype dt;
    knng_metric metric;
    const float* Xn;
    uint64_t seed;
    int64_t boundary = -1;
    bool sqn_ready = false;   // L.sqn holds the exact squared norms of X
    int update = 0;           // option "update" at bind time
    int64_t xrows = -1;       // rows of X (ids the samples may hold); -1: D.n
    void* sqn_ext = nullptr;  // squared norms of all xrows rows (distributed refine), else L.sqn
    int sms = 148;            // SM count of the current device (persistent grids)

    Run(Ctx& ctx) : c(ctx) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
            sms = 148;
        cudaGetLastError();
    }

    void bind(char* base, uint64_t* keys) {
        ws = base;
        G.keys = keys ? keys : reinterpret_cast<uint64_t*>(ws + L.keys);
        G.newmask = reinterpret_cast<uint32_t*>(ws + L.newmask);
        G.kth = reinterpret_cast<uint64_t*>(ws + L.kth);
        G.bcnt = reinterpret_cast<uint32_t*>(ws + L.bcnt);
        G.bucket = reinterpret_cast<uint64_t*>(ws + L.bucket);
        S.fwd = reinterpret_cast<uint32_t*>(ws + L.fwd);
        S.fcnt = reinterpret_cast<uint8_t*>(ws + L.fcnt);
        S.rcnt = reinterpret_cast<uint32_t*>(ws + L.rcnt);
        S.fpos = reinterpret_cast<uint32_t*>(ws + L.fpos);
        S.off = reinterpret_cast<uint64_t*>(ws + L.off);
        S.rsrc = reinterpret_cast<uint32_t*>(ws + L.rsrc);
        S.rstride = D.n * D.p;
        S.G = reinterpret_cast<uint32_t*>(ws + L.G);
        S.gcnt = reinterpret_cast<uint8_t*>(ws + L.gcnt);
        S.bsum = reinterpret_cast<uint64_t*>(ws + L.bsum);
        S.cand = L.has_cand ? reinterpret_cast<uint64_t*>(ws + L.cand) : nullptr;
        G.boff = S.off + 2 * (D.n + 1);
        G.kth_t = G.kth;
        update = g_opt_update.load();
        G.lock = update ? reinterpret_cast<unsigned int*>(ws + L.lock) : nullptr;
        G.imask = update ? reinterpret_cast<uint32_t*>(ws + L.imask) : nullptr;
        G.rec_tgt = nullptr;
        G.rec_key = nullptr;
        G.rec_cnt = nullptr;
        stats = reinterpret_cast<DevStats*>(ws + L.stats);
        Xn = metric == KNNG_COSINE ? reinterpret_cast<const float*>(ws + L.xnorm) : nullptr;
        if (metric == KNNG_CHI2) Xn = nullptr;
    }

    int warps_grid(int64_t items, int warps_per_block) const {
        return static_cast<int>((items + warps_per_block - 1) / warps_per_block);
    }

    bool zero_state() {
        if (c.err != cudaSuccess) return false;
        cudaMemsetAsync(G.bcnt, 0, static_cast<size_t>(D.n) * 4, c.stream);
        cudaMemsetAsync(S.rcnt, 0, static_cast<size_t>(2) * D.n * 4, c.stream);
        // k_rev_select loads whole forward rows ahead of their counts (the
        // entries past the count are discarded): keep them initialised
        cudaMemsetAsync(S.fwd, 0xFF, static_cast<size_t>(2) * D.n * D.p * 4, c.stream);
        // likewise the joins' planning warps copy whole sample rows (cap ids)
        cudaMemsetAsync(S.G, 0xFF, static_cast<size_t>(2) * D.n * D.cap * 4, c.stream);
        cudaMemsetAsync(stats, 0, sizeof(DevStats) * kMaxIters, c.stream);
        if (G.lock) {
            const int segs = D.k > 32 ? D.k / 32 : 1;
            cudaMemsetAsync(G.lock, 0, static_cast<size_t>(D.n) * segs * 4, c.stream);
            cudaMemsetAsync(G.imask, 0, static_cast<size_t>(D.n) * segs * 4, c.stream);
        }
        return true;
    }

    // cosine: normalised copy of the rows (D6); KNNG_E_DOMAIN on a zero row.
    // chi-square: KNNG_E_DOMAIN on a negative value; uint8 rows are copied
    // to float (D39)
    knng_status normalize() {
        if (metric == KNNG_L2SQ) return KNNG_OK;
        int* flag = reinterpret_cast<int*>(ws + L.flag);
        cudaMemsetAsync(flag, 0, 4, c.stream);
        if (metric == KNNG_COSINE) {
            c.launch("k_normalize", [&] {
                k_normalize<<<static_cast<int>((D.n + 255) / 256), 256, 0, c.stream>>>(
                    static_cast<const float*>(X), D.n, D.d, const_cast<float*>(Xn), flag);
            });
        } else if (dt == KNNG_F32) {
            c.launch("k_check_nonneg", [&] {
                k_check_nonneg<<<4 * sms, 256, 0, c.stream>>>(static_cast<const float*>(X), D.n * D.d, flag);
            });
        } else {
            float* xf = reinterpret_cast<float*>(ws + L.xnorm);
            c.launch("k_u8_to_f32", [&] {
                k_u8_to_f32<<<4 * sms, 256, 0, c.stream>>>(static_cast<const uint8_t*>(X), D.n * D.d, xf);
            });
            X = xf;
            dt = KNNG_F32;
        }
        int h = 0;
        cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, c.stream);
        const cudaError_t e = cudaStreamSynchronize(c.stream);
        if (c.err == cudaSuccess && e != cudaSuccess) {
            c.err = e;
            c.err_where = "normalize";
        }
        if (c.err != cudaSuccess) return KNNG_OK;  // reported by finish()
        if (h && metric == KNNG_COSINE) return fail(KNNG_E_DOMAIN, "zero vector under the cosine metric");
        if (h) return fail(KNNG_E_DOMAIN, "negative value under the chi-square metric");
        return KNNG_OK;
    }

    // Option exact_u8: float32 L2 input whose values are all integers in
    // [0, 255] with d <= 258 is built on an exact uint8 copy.  Every squared
    // difference and every partial sum is then an integer < 2^24, so the
    // canonical fp32 accumulation (D5) is exact and equals the integer sum:
    // the graph is bit-identical, with a quarter of the gather bytes.
    void compress() {
        g_last_exact_u8 = 0;
        if (!(metric == KNNG_L2SQ && dt == KNNG_F32 && L.xu8 && D.d <= 258 && g_opt_exact_u8.load()))
            return;
        if (c.err != cudaSuccess) return;
        int* flag = reinterpret_cast<int*>(ws + L.flag);
        const int64_t total = D.n * D.d;
        cudaMemsetAsync(flag, 0, 4, c.stream);
        uint8_t* xu8 = reinterpret_cast<uint8_t*>(ws + L.xu8);
        if (KNNG_FUSED_U8 && D.d % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && xrows < 0 && !sqn_ext) {
            // check, convert and the exact squared norms in one pass
            int* sqn = reinterpret_cast<int*>(ws + L.sqn);
            c.launch("k_to_u8", [&] {
                k_to_u8_checked<<<8 * sms, 256, 0, c.stream>>>(static_cast<const float*>(X), D.n, D.d, xu8, sqn, flag);
            });
            int h = 1;
            cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, c.stream);
            if (cudaStreamSynchronize(c.stream) != cudaSuccess || h) return;
            X = xu8;
            dt = KNNG_U8;
            sqn_ready = true;
            g_last_exact_u8 = 1;
            return;
        }
        c.launch("k_check_u8", [&] {
            k_check_u8<<<4 * sms, 256, 0, c.stream>>>(static_cast<const float*>(X), total, flag);
        });
        int h = 1;
        cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, c.stream);
        if (cudaStreamSynchronize(c.stream) != cudaSuccess || h) return;
        c.launch("k_to_u8", [&] {
            k_to_u8<<<4 * sms, 256, 0, c.stream>>>(static_cast<const float*>(X), total, xu8);
        });
        X = xu8;
        dt = KNNG_U8;
        g_last_exact_u8 = 1;
    }

    int segs() const { return D.k > 32 ? D.k / 32 : 1; }

    template <int SEG>
    void init_seg(int grid, int wpb) {
        const size_t sm = static_cast<size_t>(wpb) * 32 * 4;
        if (metric == KNNG_COSINE)
            k_init_seg<float, kMetCos, SEG><<<grid, wpb * 32, sm, c.stream>>>(nullptr, Xn, D, seed, G);
        else if (metric == KNNG_CHI2)
            k_init_seg<float, kMetChi2, SEG><<<grid, wpb * 32, sm, c.stream>>>(static_cast<const float*>(X), nullptr, D, seed, G);
        else if (dt == KNNG_F32)
            k_init_seg<float, kMetL2, SEG><<<grid, wpb * 32, sm, c.stream>>>(static_cast<const float*>(X), nullptr, D, seed, G);
        else
            k_init_seg<uint8_t, kMetL2, SEG><<<grid, wpb * 32, sm, c.stream>>>(static_cast<const uint8_t*>(X), nullptr, D, seed, G);
    }

    // with_sample: fuse the first iteration's sampling step into k_init
    // (one-segment lists, local reverse counts; iteration 0 then skips it)
    bool init_sampled = false;
    void init(bool with_sample = false) {
        const int wpb = 8;
        const int grid = warps_grid(D.n, wpb);
        const int do_sample = with_sample && KNNG_FUSED_INIT && segs() == 1 && S.fpos != nullptr && !G.imask ? 1 : 0;
        init_sampled = do_sample != 0;
        if (segs() > 1) {  // segmented lists (D40)
            c.launch("k_init", [&] {
                if (segs() == 2) init_seg<2>(grid, wpb);
                else if (segs() == 3) init_seg<3>(grid, wpb);
                else init_seg<4>(grid, wpb);
            });
            return;
        }
        c.launch("k_init", [&] {
            if (metric == KNNG_COSINE)
                k_init<float, true><<<grid, wpb * 32, wpb * 32 * 4, c.stream>>>(nullptr, Xn, D, seed, G, S, do_sample);
            else if (metric == KNNG_CHI2)
                k_init<float, kMetChi2><<<grid, wpb * 32, wpb * 32 * 4, c.stream>>>(static_cast<const float*>(X), nullptr, D, seed, G, S, do_sample);
            else if (dt == KNNG_F32)
                k_init<float, false><<<grid, wpb * 32, wpb * 32 * 4, c.stream>>>(static_cast<const float*>(X), nullptr, D, seed, G, S, do_sample);
            else
                k_init<uint8_t, false><<<grid, wpb * 32, wpb * 32 * 4, c.stream>>>(static_cast<const uint8_t*>(X), nullptr, D, seed, G, S, do_sample);
        });
    }

    // prev_iter: index of the iteration whose buckets are merged (-1: none)
    void merge_sample(int do_merge, int do_sample, int prev_iter) {
        const int wpb = 8;
        const int grid = warps_grid(D.n, wpb);
        DevStats* ps = prev_iter >= 0 ? stats + prev_iter : nullptr;
        const int sg = segs();
        c.launch(do_sample ? "k_merge_sample" : "k_merge", [&] {
            const size_t sm = static_cast<size_t>(wpb) * (sg * 32 + 32) * sizeof(uint64_t);
            if (sg == 2) k_merge_sample_seg<2><<<grid, wpb * 32, sm, c.stream>>>(D, G, S, do_merge, do_sample, ps);
            else if (sg == 3) k_merge_sample_seg<3><<<grid, wpb * 32, sm, c.stream>>>(D, G, S, do_merge, do_sample, ps);
            else if (sg == 4) k_merge_sample_seg<4><<<grid, wpb * 32, sm, c.stream>>>(D, G, S, do_merge, do_sample, ps);
            else k_merge_sample<<<grid, wpb * 32, wpb * 80 * sizeof(uint64_t), c.stream>>>(D, G, S, do_merge, do_sample, ps);
        });
    }

    // segment-major state -> merged list: ids/dists and/or keys/flags
    void export_seg(uint32_t* ids, float* dists, uint64_t* keys_out, uint8_t* flags_out) {
        const int sg = segs(), wpb = 8, grid = warps_grid(D.n, wpb);
        const size_t sm = static_cast<size_t>(wpb) * sg * 32 * 8;
        c.launch("k_export", [&] {
            if (sg == 2) k_export_seg<2><<<grid, wpb * 32, sm, c.stream>>>(D, G, ids, dists, keys_out, flags_out);
            else if (sg == 3) k_export_seg<3><<<grid, wpb * 32, sm, c.stream>>>(D, G, ids, dists, keys_out, flags_out);
            else k_export_seg<4><<<grid, wpb * 32, sm, c.stream>>>(D, G, ids, dists, keys_out, flags_out);
        });
    }
    void state_in(const uint64_t* keys_in, const uint8_t* flags) {
        const int sg = segs(), wpb = 8, grid = warps_grid(D.n, wpb);
        if (sg == 1) {
            c.launch("k_state_in", [&] { k_state_in<<<grid, 256, 0, c.stream>>>(D, G, flags); });
            return;
        }
        const size_t sm = static_cast<size_t>(wpb) * sg * (32 * 8 + 4);
        c.launch("k_state_in", [&] {
            if (sg == 2) k_state_in_seg<2><<<grid, wpb * 32, sm, c.stream>>>(D, G, keys_in, flags);
            else if (sg == 3) k_state_in_seg<3><<<grid, wpb * 32, sm, c.stream>>>(D, G, keys_in, flags);
            else k_state_in_seg<4><<<grid, wpb * 32, sm, c.stream>>>(D, G, keys_in, flags);
        });
    }
    void state_out(uint64_t* keys_out, uint8_t* flags) {
        if (segs() > 1) {
            // the merged list is written to a scratch copy first: keys_out may
            // be the buffer the segment-major state lives in
            void* tmp = nullptr;
            if (cudaMallocAsync(&tmp, static_cast<size_t>(D.n) * D.k * 8, c.stream) != cudaSuccess) {
                cudaGetLastError();
                c.err = cudaErrorMemoryAllocation;
                c.err_where = "state export";
                return;
            }
            export_seg(nullptr, nullptr, static_cast<uint64_t*>(tmp), flags);
            cudaMemcpyAsync(keys_out, tmp, static_cast<size_t>(D.n) * D.k * 8, cudaMemcpyDeviceToDevice, c.stream);
            cudaFreeAsync(tmp, c.stream);
            return;
        }
        c.launch("k_state_out", [&] {
            k_state_out<<<static_cast<int>((D.n * D.k + 255) / 256), 256, 0, c.stream>>>(D, G, flags);
        });
    }

    void reverse(uint32_t tword) {
        const int64_t nb = scan_blocks(D.n);
        c.launch("k_scan_reduce", [&] {
            k_scan_reduce<<<dim3(static_cast<unsigned>(nb), 3), kScanBlock, 0, c.stream>>>(S, D.n, nb);
        });
        c.launch("k_scan_bsums", [&] { k_scan_bsums<<<3, kScanBlock, 0, c.stream>>>(S.bsum, nb); });
        c.launch("k_scan_final", [&] {
            k_scan_final<<<dim3(static_cast<unsigned>(nb), 3), kScanBlock, 0, c.stream>>>(S, D.n, nb);
        });
        const int64_t items = D.n * D.p;
        c.launch("k_rev_scatter", [&] {
            if (D.p % 4 == 0 && g_rev_scatter4)
                k_rev_scatter4<<<dim3(static_cast<unsigned>((items / 4 + 255) / 256), 2), 256, 0, c.stream>>>(D, S);
            else
                k_rev_scatter<<<dim3(static_cast<unsigned>((items + 255) / 256), 2), 256, 0, c.stream>>>(D, S);
        });
        const int wpb = 8;
        c.launch("k_rev_select", [&] {
            k_rev_select<<<warps_grid(D.n, wpb), wpb * 32, wpb * 64 * sizeof(uint32_t), c.stream>>>(D, S, tword, seed);
        });
    }

    // returns true when the candidates were filed inside the join kernel
    bool join(int iter) {
        const int64_t batches = (D.n + kJoinNodes - 1) / kJoinNodes;
        const int grid = static_cast<int>(batches < 8ll * sms ? batches : 8ll * sms);
        DevStats* st = stats + iter;
        const size_t esz = (metric == KNNG_COSINE || dt == KNNG_F32) ? 4 : 1;
        const uintptr_t base = metric == KNNG_COSINE ? reinterpret_cast<uintptr_t>(Xn) : reinterpret_cast<uintptr_t>(X);
        const int al = ((static_cast<size_t>(D.d) * esz) % 16 == 0 && base % 16 == 0) ? 1 : 0;
        constexpr int NB = kJoinNodes;
        const int jk = g_opt_join_kernel.load();
        const bool force_v3 = jk == 1;
        if (update) {
            // the paper's immediate update under spinlocks (join_locked.cuh):
            // GNND-r1 (full), GNND (segment locks), GNND-r2 (one lock)
            const int one = update == 3;
            const int g2 = static_cast<int>(D.n < 16ll * sms * 32 ? D.n : 16ll * sms * 32);
            c.launch("k_join", [&] {
                if (metric == KNNG_COSINE) {
                    if (update == 1) k_join_locked<float, kMetCos, true><<<g2, kLkThreads, 0, c.stream>>>(nullptr, Xn, D, G, S, boundary, one, st);
                    else k_join_locked<float, kMetCos, false><<<g2, kLkThreads, 0, c.stream>>>(nullptr, Xn, D, G, S, boundary, one, st);
                } else if (metric == KNNG_CHI2) {
                    const float* Xf = static_cast<const float*>(X);
                    if (update == 1) k_join_locked<float, kMetChi2, true><<<g2, kLkThreads, 0, c.stream>>>(Xf, nullptr, D, G, S, boundary, one, st);
                    else k_join_locked<float, kMetChi2, false><<<g2, kLkThreads, 0, c.stream>>>(Xf, nullptr, D, G, S, boundary, one, st);
                } else if (dt == KNNG_F32) {
                    const float* Xf = static_cast<const float*>(X);
                    if (update == 1) k_join_locked<float, kMetL2, true><<<g2, kLkThreads, 0, c.stream>>>(Xf, nullptr, D, G, S, boundary, one, st);
                    else k_join_locked<float, kMetL2, false><<<g2, kLkThreads, 0, c.stream>>>(Xf, nullptr, D, G, S, boundary, one, st);
                } else {
                    const uint8_t* Xu = static_cast<const uint8_t*>(X);
                    if (update == 1) k_join_locked<uint8_t, kMetL2, true><<<g2, kLkThreads, 0, c.stream>>>(Xu, nullptr, D, G, S, boundary, one, st);
                    else k_join_locked<uint8_t, kMetL2, false><<<g2, kLkThreads, 0, c.stream>>>(Xu, nullptr, D, G, S, boundary, one, st);
                }
            });
            return true;
        }
        const bool u8_slab = al && metric == KNNG_L2SQ && dt == KNNG_U8 && D.d <= kTcRowBytes && D.d % 16 == 0;
        if (u8_slab && jk == 0) {
            // uint8 rows of one 128-B slab: Gram tiles on the tensor cores
            int* sqn = static_cast<int*>(sqn_ext ? sqn_ext : ws + L.sqn);
            const int64_t xr = xrows >= 0 ? xrows : D.n;
            if (!sqn_ready) {
                c.launch("k_sqnorm_u8", [&] {
                    k_sqnorm_u8<<<static_cast<int>((xr + 255) / 256), 256, 0, c.stream>>>(
                        static_cast<const uint8_t*>(X), xr, D.d, sqn);
                });
                sqn_ready = true;
            }
            unsigned long long* work = reinterpret_cast<unsigned long long*>(ws + L.flag + 8);
            cudaMemsetAsync(work, 0, 8, c.stream);
            c.launch("k_join", [&] {
                constexpr size_t sm = TcCfg::kSmem;
                CUtensorMap tm;
                memset(&tm, 0, sizeof(tm));
                // rows by TMA gather4; 16-B cp.async copies if the driver's
                // tensor-map encoder is unavailable (bit-identical)
                const bool tma = make_row_tmap(X, xr, D.d, &tm);
                const bool rec = G.rec_cnt != nullptr;  // record mode: the distributed refine
                auto go = [&](auto kfn) {
                    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                    kfn<<<3 * sms, 9 * 32, sm, c.stream>>>(static_cast<const uint8_t*>(X), sqn, D, G, S, boundary,
                                                          work, st, tm);
                };
                // 8 epilogue warps, 3 CTAs per SM
                if (tma) rec ? go(k_join_tc<8, 3, true, true>) : go(k_join_tc<8, 3, true, false>);
                else rec ? go(k_join_tc<8, 3, false, true>) : go(k_join_tc<8, 3, false, false>);
            });
            return true;
        }
        const bool f32_tc = al && metric != KNNG_CHI2 && (metric == KNNG_COSINE || dt == KNNG_F32) && D.d % 4 == 0 && D.d <= 128;
        if (f32_tc && jk == 4) {
            // float rows: TF32 Gram tiles on the tensor cores, exact selection
            // by canonical recomputation inside the error-bound window.  Opt-in:
            // on DEEP-shaped rows it measured 36.6 ms per launch against 12.0 ms
            // for the CUDA-core join (profiles/r01s2_ncu_k_join_tcf_deep.txt),
            // so the automatic choice stays on k_join_ws for float rows.
            const float* Xf = metric == KNNG_COSINE ? Xn : static_cast<const float*>(X);
            float* sqn = static_cast<float*>(sqn_ext ? sqn_ext : ws + L.sqn);
            const int64_t xr = xrows >= 0 ? xrows : D.n;
            if (!sqn_ready) {
                c.launch("k_sqnorm_f32", [&] {
                    k_sqnorm_f32<<<static_cast<int>((xr + 255) / 256), 256, 0, c.stream>>>(Xf, xr, D.d, sqn);
                });
                sqn_ready = true;
            }
            unsigned long long* work = reinterpret_cast<unsigned long long*>(ws + L.flag + 8);
            cudaMemsetAsync(work, 0, 8, c.stream);
            c.launch("k_join", [&] {
                const int ka = (D.d + 31) / 32;
                const bool cs = metric == KNNG_COSINE;
                auto go = [&](auto kfn, size_t sm, int ctas) {
                    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                    kfn<<<ctas * sms, kTcThreads, sm, c.stream>>>(Xf, sqn, D, G, S, boundary, work, st);
                };
                if (ka == 1) cs ? go(k_join_tcf<1, true>, TcfCfg<1>::kSmem, TcfCfg<1>::kCtas)
                                : go(k_join_tcf<1, false>, TcfCfg<1>::kSmem, TcfCfg<1>::kCtas);
                else if (ka == 2) cs ? go(k_join_tcf<2, true>, TcfCfg<2>::kSmem, TcfCfg<2>::kCtas)
                                     : go(k_join_tcf<2, false>, TcfCfg<2>::kSmem, TcfCfg<2>::kCtas);
                else if (ka == 3) cs ? go(k_join_tcf<3, true>, TcfCfg<3>::kSmem, TcfCfg<3>::kCtas)
                                     : go(k_join_tcf<3, false>, TcfCfg<3>::kSmem, TcfCfg<3>::kCtas);
                else cs ? go(k_join_tcf<4, true>, TcfCfg<4>::kSmem, TcfCfg<4>::kCtas)
                        : go(k_join_tcf<4, false>, TcfCfg<4>::kSmem, TcfCfg<4>::kCtas);
            });
            return true;
        }
        if (al && !force_v3) {
            // warp-specialised pipeline (bulk row copies need 16-B aligned,
            // 16-B multiple row slabs)
#ifndef WS_STG
#define WS_STG 3
#endif
#ifndef WS_STP
#define WS_STP 2
#endif
            // Fewer stages are faster: the shared memory they leave to L1
            // serves the row gathers (rows recur across nearby batches) --
            // DEEP 1M packed: 10.1 (4 stages) -> 9.2 (3) -> 9.1 ms (2);
            // scalar: 10.4 (5) -> 9.7 (4) -> 9.65 ms (3)
            // (tools/ws_stage_variants.sh, profiles/r02_float_join_ab.txt)
            constexpr int STG = WS_STG;  // 32-KB stages (row-slab layout: u8 and the scalar float tile)
            constexpr int STP = WS_STP;  // 33-KB stages (pair-interleaved layout of the packed FP32x2 tile)
            // float tile: the packed FP32x2 tile for L2 (DEEP-shaped 9.1 vs
            // 9.65 ms per launch, GIST-shaped 10.4 vs 11.8 ms) and
            // chi-square, the scalar tile for cosine (8.1 vs 8.5 ms: its
            // one FMA per dimension leaves the packed tile no issue slots to
            // save) -- profiles/r02_float_join_ab.txt.  Options 2 / 3 force one.
            const bool pk = jk == 2 || (jk != 3 && metric != KNNG_COSINE);
            unsigned long long* work = reinterpret_cast<unsigned long long*>(ws + L.flag + 8);
            cudaMemsetAsync(work, 0, 8, c.stream);
            const float* Xf = static_cast<const float*>(X);
            auto go = [&](auto kfn, size_t sm, auto Xp, const float* Xnp) {
                cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                kfn<<<sms, kWsThreads, sm, c.stream>>>(Xp, Xnp, D, G, S, boundary, work, st);
            };
            c.launch("k_join", [&] {
                if (metric == KNNG_COSINE) {
                    if (pk) go(k_join_ws<float, kMetCos, STP, true>, WsCfg<float, kMetCos, STP, true>::kSmem, Xf, Xn);
                    else go(k_join_ws<float, kMetCos, STG, false>, WsCfg<float, kMetCos, STG, false>::kSmem, Xf, Xn);
                } else if (metric == KNNG_CHI2) {
                    go(k_join_ws<float, kMetChi2, STP, true>, WsCfg<float, kMetChi2, STP, true>::kSmem, Xf, nullptr);
                } else if (dt == KNNG_F32) {
                    if (pk) go(k_join_ws<float, kMetL2, STP, true>, WsCfg<float, kMetL2, STP, true>::kSmem, Xf, nullptr);
                    else go(k_join_ws<float, kMetL2, STG, false>, WsCfg<float, kMetL2, STG, false>::kSmem, Xf, nullptr);
                } else {
                    go(k_join_ws<uint8_t, kMetL2, STG, false>, WsCfg<uint8_t, kMetL2, STG, false>::kSmem,
                       static_cast<const uint8_t*>(X), nullptr);
                }
            });
            return true;
        }
        if (!S.cand) {  // legacy join on rows the workspace did not plan it for
            void* p = nullptr;
            if (cudaMallocAsync(&p, static_cast<size_t>(D.n) * 3 * D.cap * 8, c.stream) != cudaSuccess) {
                cudaGetLastError();
                c.err = cudaErrorMemoryAllocation;
                c.err_where = "join staging allocation";
                return true;
            }
            c.owned_extra = p;
            S.cand = static_cast<uint64_t*>(p);
        }
        c.launch("k_join", [&] {
            if (metric == KNNG_COSINE) {
                constexpr size_t sm = join_smem_bytes<float, true, NB>();
                cudaFuncSetAttribute(k_join<float, true, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                k_join<float, true, NB><<<grid, NB * 64, sm, c.stream>>>(nullptr, Xn, D, S, boundary, al, st);
            } else if (metric == KNNG_CHI2) {
                constexpr size_t sm = join_smem_bytes<float, kMetChi2, NB>();
                cudaFuncSetAttribute(k_join<float, kMetChi2, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                k_join<float, kMetChi2, NB><<<grid, NB * 64, sm, c.stream>>>(static_cast<const float*>(X), nullptr, D, S,
                                                                            boundary, al, st);
            } else if (dt == KNNG_F32) {
                constexpr size_t sm = join_smem_bytes<float, false, NB>();
                cudaFuncSetAttribute(k_join<float, false, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                k_join<float, false, NB><<<grid, NB * 64, sm, c.stream>>>(static_cast<const float*>(X), nullptr, D, S,
                                                                         boundary, al, st);
            } else {
                constexpr size_t sm = join_smem_bytes<uint8_t, false, NB>();
                cudaFuncSetAttribute(k_join<uint8_t, false, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                k_join<uint8_t, false, NB><<<grid, NB * 64, sm, c.stream>>>(static_cast<const uint8_t*>(X), nullptr, D,
                                                                           S, boundary, al, st);
            }
        });
        return false;
    }

    void scatter(int iter) {
        const int64_t items = D.n * 3 * D.cap;
        DevStats* st = stats + iter;
        c.launch("k_cand_scatter", [&] {
            k_cand_scatter<<<static_cast<int>((items + 255) / 256), 256, 0, c.stream>>>(D, G, S, st);
        });
    }

    void iteration(int iter, uint32_t tword, bool merge_first) {
        if (!(iter == 0 && init_sampled)) merge_sample(merge_first ? 1 : 0, 1, merge_first ? iter - 1 : -1);
        reverse(tword);
        if (!join(iter)) scatter(iter);
    }

    void export_graph(uint32_t* ids, float* dists) {
        if (segs() > 1) {
            export_seg(ids, dists, nullptr, nullptr);
            return;
        }
        const int64_t total = D.n * D.k;
        c.launch("k_export", [&] {
            k_export<<<static_cast<int>((total + 255) / 256), 256, 0, c.stream>>>(G.keys, total, ids, dists);
        });
    }

    void collect_stats(int iters) {
        std::vector<DevStats> h(iters > 0 ? iters : 1);
        if (c.err == cudaSuccess && iters > 0) {
            cudaMemcpyAsync(h.data(), stats, sizeof(DevStats) * iters, cudaMemcpyDeviceToHost, c.stream);
            cudaStreamSynchronize(c.stream);
        }
        g_last_stats.clear();
        for (int i = 0; i < iters; ++i) {
            knng_iter_stats s;
            s.joins = static_cast<int64_t>(h[i].joins);
            s.sum_m = static_cast<int64_t>(h[i].sum_m);
            s.sum_q = static_cast<int64_t>(h[i].sum_q);
            s.dist_evals = static_cast<int64_t>(h[i].dist_evals);
            s.candidates = static_cast<int64_t>(h[i].candidates);
            s.appended = static_cast<int64_t>(h[i].appended);
            s.accepted = static_cast<int64_t>(h[i].accepted);
            s.rows = static_cast<int64_t>(h[i].rows);
            s.recomputed = static_cast<int64_t>(h[i].recomputed);
            g_last_stats.push_back(s);
        }
    }
};

std::atomic<bool> g_pool_ready[64];

knng_status get_workspace(Ctx& c, void* workspace, size_t bytes, size_t need, char** out) {
    if (workspace == nullptr && bytes == 0) {
        // Library-owned workspace comes from the device's default stream-
        // ordered pool; keep freed blocks reserved in the pool (release
        // threshold = max) so repeated calls do not re-map GBs of memory.
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64 && !g_pool_ready[dev].exchange(true)) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        }
        void* p = nullptr;
        const cudaError_t e = cudaMallocAsync(&p, need, c.stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(KNNG_E_NOMEM, "cannot allocate %zu bytes of workspace: %s", need, cudaGetErrorString(e));
        }
        c.owned_ws = p;
        *out = static_cast<char*>(p);
        return KNNG_OK;
    }
    if (bytes < need) return fail(KNNG_E_USAGE, "workspace too small: %zu < %zu bytes", bytes, need);
    if (!is_device_ptr(workspace)) return fail(KNNG_E_USAGE, "workspace is not a device pointer");
    // the layout holds u64 arrays, 16-B vector loads and mbarrier words
    if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
        return fail(KNNG_E_USAGE, "workspace must be 256-byte aligned");
    *out = static_cast<char*>(workspace);
    return KNNG_OK;
}

#include "dist_api.cuh"

}  // namespace

// ======================================================================
extern "C" {

size_t knng_build_workspace_bytes(knng_dtype dt, int64_t n, int32_t d, int32_t k, int32_t sample_size,
                                  knng_metric metric) {
    if (check_common(dt, n, d, k, metric, sample_size) != KNNG_OK) return 0;
    return make_layout(n, d, k, sample_size, needs_xcopy(metric, dt), true, false, dt == KNNG_F32 && metric == KNNG_L2SQ).total;
}

knng_status knng_build(const void* vectors, knng_dtype dt, int64_t n, int32_t d, int32_t k, knng_metric metric,
                       int32_t iters, int32_t sample_size, uint64_t seed, uint32_t* out_ids, float* out_dists,
                       void* workspace, size_t workspace_bytes, void* stream) {
    knng_status s = check_common(dt, n, d, k, metric, sample_size);
    if (s) return s;
    if (iters < 1 || iters > kMaxIters) return fail(KNNG_E_USAGE, "iters must be in [1, %d] (got %d)", kMaxIters, iters);
    if (!vectors || !out_ids || !out_dists) return fail(KNNG_E_USAGE, "null pointer argument");
    if (!is_device_ptr(vectors) || !is_device_ptr(out_ids) || !is_device_ptr(out_dists))
        return fail(KNNG_E_USAGE, "vectors/out_ids/out_dists must be device pointers");
    Ctx c;
    c.stream = static_cast<cudaStream_t>(stream);
    c.timing = g_timing.load() != 0;
    Run R(c);
    R.L = make_layout(n, d, k, sample_size, needs_xcopy(metric, dt), true, false, dt == KNNG_F32 && metric == KNNG_L2SQ);
    char* ws = nullptr;
    if ((s = get_workspace(c, workspace, workspace_bytes, R.L.total, &ws))) return s;
    R.D = Dims{n, d, k, sample_size, 2 * sample_size};
    R.X = vectors;
    R.dt = dt;
    R.metric = metric;
    R.seed = seed;
    R.bind(ws, nullptr);
    R.zero_state();
    if ((s = R.normalize())) return s;
    R.compress();
    R.init(true);
    for (int t = 0; t < iters; ++t) R.iteration(t, static_cast<uint32_t>(t), t > 0);
    R.merge_sample(1, 0, iters - 1);
    R.export_graph(out_ids, out_dists);
    R.collect_stats(iters);
    return c.finish();
}

knng_status knng_build_host(const void* host_vectors, knng_dtype dt, int64_t n, int32_t d, int32_t k,
                            knng_metric metric, int32_t iters, int32_t sample_size, uint64_t seed,
                            uint32_t* host_out_ids, float* host_out_dists, void* stream) {
    knng_status s = check_common(dt, n, d, k, metric, sample_size);
    if (s) return s;
    if (iters < 1 || iters > kMaxIters) return fail(KNNG_E_USAGE, "iters must be in [1, %d] (got %d)", kMaxIters, iters);
    if (!host_vectors || !host_out_ids || !host_out_dists) return fail(KNNG_E_USAGE, "null pointer argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t vbytes = static_cast<size_t>(n) * d * (dt == KNNG_F32 ? 4 : 1);
    const size_t gbytes = static_cast<size_t>(n) * k * 4;
    void *dv = nullptr, *di = nullptr, *dd = nullptr;
    cudaError_t e = cudaMallocAsync(&dv, vbytes, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&di, gbytes, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&dd, gbytes, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dv, host_vectors, vbytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
        s = knng_build(dv, dt, n, d, k, metric, iters, sample_size, seed, static_cast<uint32_t*>(di),
                       static_cast<float*>(dd), nullptr, 0, stream);
        if (s == KNNG_OK) {
            e = cudaMemcpyAsync(host_out_ids, di, gbytes, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(host_out_dists, dd, gbytes, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        }
    }
    if (dv) cudaFreeAsync(dv, st);
    if (di) cudaFreeAsync(di, st);
    if (dd) cudaFreeAsync(dd, st);
    cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? KNNG_E_NOMEM : KNNG_E_CUDA, "knng_build_host: %s",
                    cudaGetErrorString(e));
    }
    return s;
}

knng_status knng_bruteforce(const void* vectors, knng_dtype dt, int64_t n, int32_t d, knng_metric metric,
                            const int64_t* queries, int64_t nq, int32_t kq, uint32_t* out_ids, float* out_dists,
                            void* stream) {
    if (dt != KNNG_F32 && dt != KNNG_U8) return fail(KNNG_E_USAGE, "unknown dtype");
    if (metric != KNNG_L2SQ && metric != KNNG_COSINE && metric != KNNG_CHI2) return fail(KNNG_E_USAGE, "unknown metric");
    if (metric == KNNG_COSINE && dt != KNNG_F32) return fail(KNNG_E_USAGE, "cosine requires float32 vectors");
    if (kq < 1 || kq > 32 || n <= kq || d < 1 || nq < 0) return fail(KNNG_E_USAGE, "bad bruteforce arguments");
    if (nq == 0) return KNNG_OK;
    if (!is_device_ptr(vectors) || !is_device_ptr(queries) || !is_device_ptr(out_ids) || !is_device_ptr(out_dists))
        return fail(KNNG_E_USAGE, "bruteforce arguments must be device pointers");
    Ctx c;
    c.stream = static_cast<cudaStream_t>(stream);
    c.timing = g_timing.load() != 0;
    const bool cosine = metric == KNNG_COSINE, chi2 = metric == KNNG_CHI2;
    const size_t esz = (cosine || chi2 || dt == KNNG_F32) ? 4 : 1;
    const size_t outb = static_cast<size_t>(nq) * kq * 8;
    const size_t xnb = needs_xcopy(metric, dt) ? static_cast<size_t>(n) * d * 4 : 0;
    char* ws = nullptr;
    knng_status s;
    if ((s = get_workspace(c, nullptr, 0, align_up(outb) + align_up(xnb) + 256, &ws))) return s;
    uint64_t* keys = reinterpret_cast<uint64_t*>(ws);
    float* Xn = xnb ? reinterpret_cast<float*>(ws + align_up(outb)) : nullptr;
    int* flag = reinterpret_cast<int*>(ws + align_up(outb) + align_up(xnb));
    const float* Xf = static_cast<const float*>(vectors);  // chi-square rows (float)
    if (chi2) {
        cudaMemsetAsync(flag, 0, 4, c.stream);
        if (dt == KNNG_U8) {
            c.launch("k_u8_to_f32", [&] {
                k_u8_to_f32<<<592, 256, 0, c.stream>>>(static_cast<const uint8_t*>(vectors), n * d, Xn);
            });
            Xf = Xn;
        } else {
            c.launch("k_check_nonneg", [&] { k_check_nonneg<<<592, 256, 0, c.stream>>>(Xf, n * d, flag); });
            int h = 0;
            cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, c.stream);
            cudaStreamSynchronize(c.stream);
            if (h) return fail(KNNG_E_DOMAIN, "negative value under the chi-square metric");
        }
    }
    if (cosine) {
        cudaMemsetAsync(flag, 0, 4, c.stream);
        c.launch("k_normalize", [&] {
            k_normalize<<<static_cast<int>((n + 255) / 256), 256, 0, c.stream>>>(static_cast<const float*>(vectors), n,
                                                                                 d, Xn, flag);
        });
        int h = 0;
        cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        if (h) return fail(KNNG_E_DOMAIN, "zero vector under the cosine metric");
    }
    int W = 8;
    const int stride = esz == 4 ? bf_stride_elems<float>(d) : bf_stride_elems<uint8_t>(d);
    auto smem_for = [&](int w) {
        return static_cast<size_t>(32 + w * kBfQPerWarp) * stride * esz + static_cast<size_t>(w) * 32 * sizeof(Elem);
    };
    while (W > 1 && smem_for(W) > 200 * 1024) W >>= 1;
    const size_t smem = smem_for(W);
    if (smem > 220 * 1024) return fail(KNNG_E_USAGE, "d too large for the brute-force kernel");
    const int64_t per_block = static_cast<int64_t>(W) * kBfQPerWarp;
    const int grid = static_cast<int>((nq + per_block - 1) / per_block);
    c.launch("k_bruteforce", [&] {
        if (cosine) {
            cudaFuncSetAttribute(k_bruteforce<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k_bruteforce<float, true><<<grid, W * 32, smem, c.stream>>>(nullptr, Xn, n, d, queries, nq, kq, keys);
        } else if (chi2) {
            cudaFuncSetAttribute(k_bruteforce<float, kMetChi2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k_bruteforce<float, kMetChi2><<<grid, W * 32, smem, c.stream>>>(Xf, nullptr, n, d, queries, nq, kq, keys);
        } else if (dt == KNNG_F32) {
            cudaFuncSetAttribute(k_bruteforce<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k_bruteforce<float, false><<<grid, W * 32, smem, c.stream>>>(static_cast<const float*>(vectors), nullptr, n, d,
                                                                          queries, nq, kq, keys);
        } else {
            cudaFuncSetAttribute(k_bruteforce<uint8_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k_bruteforce<uint8_t, false><<<grid, W * 32, smem, c.stream>>>(static_cast<const uint8_t*>(vectors), nullptr, n,
                                                                            d, queries, nq, kq, keys);
        }
    });
    const int64_t total = nq * kq;
    c.launch("k_export", [&] {
        k_export<<<static_cast<int>((total + 255) / 256), 256, 0, c.stream>>>(keys, total, out_ids, out_dists);
    });
    return c.finish();
}

// ------------------------------------------------------------ debug ABI
knng_status knng_debug_init(const void* vectors, knng_dtype dt, int64_t n, int32_t d, int32_t k,
                            knng_metric metric, uint64_t seed, uint64_t* keys, uint8_t* flags, void* stream) {
    knng_status s = check_common(dt, n, d, k, metric, 1);
    if (s) return s;
    if (!is_device_ptr(vectors) || !is_device_ptr(keys) || !is_device_ptr(flags))
        return fail(KNNG_E_USAGE, "arguments must be device pointers");
    Ctx c;
    c.stream = static_cast<cudaStream_t>(stream);
    c.timing = g_timing.load() != 0;
    Run R(c);
    R.L = make_layout(n, d, k, 1, needs_xcopy(metric, dt), false, false, dt == KNNG_F32 && metric == KNNG_L2SQ);
    char* ws = nullptr;
    if ((s = get_workspace(c, nullptr, 0, R.L.total, &ws))) return s;
    R.D = Dims{n, d, k, 1, 2};
    R.X = vectors;
    R.dt = dt;
    R.metric = metric;
    R.seed = seed;
    R.bind(ws, keys);
    if ((s = R.normalize())) return s;
    R.compress();
    R.init();
    R.state_out(keys, flags);
    return c.finish();
}

knng_status knng_debug_iterate(const void* vectors, knng_dtype dt, int64_t n, int32_t d, int32_t k,
                               knng_metric metric, int32_t sample_size, uint32_t tword, uint64_t seed,
                               int64_t boundary, uint64_t* keys, uint8_t* flags, knng_iter_stats* host_stats,
                               void* workspace, size_t workspace_bytes, void* stream) {
    knng_status s = check_common(dt, n, d, k, metric, sample_size);
    if (s) return s;
    if (!is_device_ptr(vectors) || !is_device_ptr(keys) || !is_device_ptr(flags))
        return fail(KNNG_E_USAGE, "arguments must be device pointers");
    Ctx c;
    c.stream = static_cast<cudaStream_t>(stream);
    c.timing = g_timing.load() != 0;
    Run R(c);
    R.L = make_layout(n, d, k, sample_size, needs_xcopy(metric, dt), false, false, dt == KNNG_F32 && metric == KNNG_L2SQ);
    char* ws = nullptr;
    if ((s = get_workspace(c, workspace, workspace_bytes, R.L.total, &ws))) return s;
    R.D = Dims{n, d, k, sample_size, 2 * sample_size};
    R.X = vectors;
    R.dt = dt;
    R.metric = metric;
    R.seed = seed;
    R.boundary = boundary;
    R.bind(ws, keys);
    R.zero_state();
    if ((s = R.normalize())) return s;
    R.compress();
    R.state_in(keys, flags);
    R.iteration(0, tword, false);
    R.merge_sample(1, 0, 0);
    R.state_out(keys, flags);
    R.collect_stats(1);
    if (host_stats && !g_last_stats.empty()) *host_stats = g_last_stats[0];
    return c.finish();
}

knng_status knng_debug_sample(int64_t n, int32_t k, int32_t sample_size, uint32_t tword, uint64_t seed,
                              const uint64_t* keys, const uint8_t* flags, uint32_t* Gn, int32_t* cn, uint32_t* Go,
                              int32_t* co, void* workspace, size_t workspace_bytes, void* stream) {
    knng_status s = check_common(KNNG_F32, n, 1, k, KNNG_L2SQ, sample_size);
    if (s) return s;
    if (!is_device_ptr(keys) || !is_device_ptr(flags) || !is_device_ptr(Gn) || !is_device_ptr(cn) ||
        !is_device_ptr(Go) || !is_device_ptr(co))
        return fail(KNNG_E_USAGE, "arguments must be device pointers");
    Ctx c;
    c.stream = static_cast<cudaStream_t>(stream);
    Run R(c);
    R.L = make_layout(n, 1, k, sample_size, false, true, false);
    char* ws = nullptr;
    if ((s = get_workspace(c, workspace, workspace_bytes, R.L.total, &ws))) return s;
    R.D = Dims{n, 1, k, sample_size, 2 * sample_size};
    R.metric = KNNG_L2SQ;
    R.seed = seed;
    R.bind(ws, nullptr);
    R.zero_state();
    cudaMemcpyAsync(R.G.keys, keys, static_cast<size_t>(n) * k * 8, cudaMemcpyDeviceToDevice, c.stream);
    R.state_in(R.G.keys, flags);
    R.merge_sample(0, 1, -1);
    R.reverse(tword);
    c.launch("k_samples_out", [&] {
        k_samples_out<<<static_cast<int>((n * R.D.cap + 255) / 256), 256, 0, c.stream>>>(R.D, R.S, Gn, cn, Go, co);
    });
    return c.finish();
}

knng_status knng_debug_philox(const uint32_t* ctr, int64_t m, uint64_t seed, uint32_t* out, void* stream) {
    if (m < 0) return fail(KNNG_E_USAGE, "m < 0");
    if (m == 0) return KNNG_OK;
    if (!is_device_ptr(ctr) || !is_device_ptr(out)) return fail(KNNG_E_USAGE, "arguments must be device pointers");
    Ctx c;
    c.stream = static_cast<cudaStream_t>(stream);
    c.launch("k_philox_test", [&] {
        k_philox_test<<<static_cast<int>((m + 255) / 256), 256, 0, c.stream>>>(ctr, m, seed, out);
    });
    return c.finish();
}

// ------------------------------------------------------------ GGM (Alg. 3)
size_t knng_merge_workspace_bytes(knng_dtype dt, int64_t nA, int64_t nB, int32_t d, int32_t k, int32_t sample_size,
                                  knng_metric metric) {
    if (check_common(dt, nA + nB, d, k, metric, sample_size) != KNNG_OK) return 0;
    const int64_t n = nA + nB;
    const size_t vbytes = static_cast<size_t>(n) * d * (dt == KNNG_F32 ? 4 : 1);
    return make_layout(n, d, k, sample_size, needs_xcopy(metric, dt), true, true, dt == KNNG_F32 && metric == KNNG_L2SQ).total + align_up(vbytes);
}

knng_status knng_merge(const void* vecA, int64_t nA, const uint32_t* idsA, const float* distsA, const void* vecB,
                       int64_t nB, const uint32_t* idsB, const float* distsB, knng_dtype dt, int32_t d, int32_t k,
                       knng_metric metric, int32_t merge_iters, int32_t sample_size, int32_t level, uint64_t seed,
                       uint32_t* out_ids, float* out_dists, void* workspace, size_t workspace_bytes, void* stream) {
    const int64_t n = nA + nB;
    knng_status s = check_common(dt, n, d, k, metric, sample_size);
    if (s) return s;
    if (k > 32) return fail(KNNG_E_USAGE, "GGM merges one-segment lists (k <= 32)");
    const int kr = k / 2;
    if (nA < kr || nB < kr || nA < 1 || nB < 1)
        return fail(KNNG_E_USAGE, "each graph needs at least floor(k/2) = %d nodes (nA=%lld, nB=%lld)", kr,
                    static_cast<long long>(nA), static_cast<long long>(nB));
    if (nA <= k || nB <= k) return fail(KNNG_E_USAGE, "each input graph needs n > k");
    if (merge_iters < 0 || merge_iters > kMaxIters) return fail(KNNG_E_USAGE, "merge_iters must be in [0, %d]", kMaxIters);
    if (level < 0 || level > 0x7FFF) return fail(KNNG_E_USAGE, "level must be in [0, 32767]");
    if (!is_device_ptr(vecA) || !is_device_ptr(vecB) || !is_device_ptr(idsA) || !is_device_ptr(distsA) ||
        !is_device_ptr(idsB) || !is_device_ptr(distsB) || !is_device_ptr(out_ids) || !is_device_ptr(out_dists))
        return fail(KNNG_E_USAGE, "arguments must be device pointers");
    Ctx c;
    c.stream = static_cast<cudaStream_t>(stream);
    c.timing = g_timing.load() != 0;
    Run R(c);
    R.L = make_layout(n, d, k, sample_size, needs_xcopy(metric, dt), true, true, dt == KNNG_F32 && metric == KNNG_L2SQ);
    const size_t esz = dt == KNNG_F32 ? 4 : 1;
    const size_t vbytes = static_cast<size_t>(n) * d * esz;
    char* ws = nullptr;
    if ((s = get_workspace(c, workspace, workspace_bytes, R.L.total + align_up(vbytes), &ws))) return s;
    // combined vector set [S1; S2] (S = S1 U S2); used in place when
    // the caller's B rows already follow A's (the sharded tree's layout)
    const char* X = static_cast<const char*>(vecA);
    if (static_cast<const char*>(vecB) != X + static_cast<size_t>(nA) * d * esz) {
        char* Xc = ws + R.L.total;
        cudaMemcpyAsync(Xc, vecA, static_cast<size_t>(nA) * d * esz, cudaMemcpyDeviceToDevice, c.stream);
        cudaMemcpyAsync(Xc + static_cast<size_t>(nA) * d * esz, vecB, static_cast<size_t>(nB) * d * esz,
                        cudaMemcpyDeviceToDevice, c.stream);
        X = Xc;
    }
    R.D = Dims{n, d, k, sample_size, 2 * sample_size};
    R.X = X;
    R.dt = dt;
    R.metric = metric;
    R.seed = seed;
    R.boundary = nA;
    R.bind(ws, nullptr);
    R.zero_state();
    if ((s = R.normalize())) return s;
    R.compress();
    uint64_t* reserved = reinterpret_cast<uint64_t*>(ws + R.L.reserved);
    const int grid = R.warps_grid(n, 8);
    int* bad = reinterpret_cast<int*>(ws + R.L.flag) + 1;
    cudaMemsetAsync(bad, 0, 4, c.stream);
    c.launch("k_ggm_seed", [&] {
        if (metric == KNNG_COSINE)
            k_ggm_seed<float, true><<<grid, 256, 256 * 4, c.stream>>>(nullptr, R.Xn, R.D, nA, level, seed, idsA, distsA, idsB,
                                                                distsB, R.G, reserved, bad);
        else if (metric == KNNG_CHI2)
            k_ggm_seed<float, kMetChi2><<<grid, 256, 256 * 4, c.stream>>>(reinterpret_cast<const float*>(R.X), nullptr, R.D, nA,
                                                                     level, seed, idsA, distsA, idsB, distsB, R.G, reserved, bad);
        else if (R.dt == KNNG_F32)
            k_ggm_seed<float, false><<<grid, 256, 256 * 4, c.stream>>>(reinterpret_cast<const float*>(R.X), nullptr, R.D, nA,
                                                                 level, seed, idsA, distsA, idsB, distsB, R.G, reserved, bad);
        else
            k_ggm_seed<uint8_t, false><<<grid, 256, 256 * 4, c.stream>>>(reinterpret_cast<const uint8_t*>(R.X), nullptr, R.D,
                                                                   nA, level, seed, idsA, distsA, idsB, distsB, R.G,
                                                                   reserved, bad);
    });
    {
        int h = 0;
        cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, c.stream);
        const cudaError_t e = cudaStreamSynchronize(c.stream);
        if (c.err == cudaSuccess && e == cudaSuccess && h)
            return fail(KNNG_E_USAGE, "input graph holds an id outside its own node range");
    }
    for (int t = 0; t < merge_iters; ++t)
        R.iteration(t, 0x80000000u | (static_cast<uint32_t>(level) << 16) | static_cast<uint32_t>(t), t > 0);
    R.merge_sample(1, 0, merge_iters - 1);
    c.launch("k_ggm_finalize", [&] {
        k_ggm_finalize<<<grid, 256, 256 * sizeof(uint64_t), c.stream>>>(R.D, R.G, reserved);
    });
    R.export_graph(out_ids, out_dists);
    R.collect_stats(merge_iters);
    return c.finish();
}

// ------------------------------------------------------------ incremental
knng_status knng_extend(const void* vec_old, int64_t n_old, const uint32_t* ids_old, const float* dists_old,
                        const void* vec_new, int64_t n_new, knng_dtype dt, int32_t d, int32_t k, knng_metric metric,
                        int32_t iters, int32_t merge_iters, int32_t sample_size, uint64_t seed, uint32_t* out_ids,
                        float* out_dists, void* stream) {
    // "As the new data come in, GNND is called to build a sub-graph on the
    // first hand.  Thereafter, GGM is called to join this new sub-graph into
    // the existing k-NN graph": knng_build on the batch, knng_merge.
    knng_status s = check_common(dt, n_new, d, k, metric, sample_size);
    if (s) return s;
    if ((s = check_common(dt, n_old + n_new, d, k, metric, sample_size))) return s;
    if (k > 32) return fail(KNNG_E_USAGE, "GGM merges one-segment lists (k <= 32)");
    if (n_old <= k) return fail(KNNG_E_USAGE, "the existing graph needs n_old > k");
    if (iters < 1 || iters > kMaxIters) return fail(KNNG_E_USAGE, "iters must be in [1, %d]", kMaxIters);
    if (!is_device_ptr(vec_new) || !is_device_ptr(out_ids) || !is_device_ptr(out_dists))
        return fail(KNNG_E_USAGE, "arguments must be device pointers");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    void *ib = nullptr, *db = nullptr;
    const size_t gb = static_cast<size_t>(n_new) * k * 4;
    if (cudaMallocAsync(&ib, gb, st) != cudaSuccess || cudaMallocAsync(&db, gb, st) != cudaSuccess) {
        cudaGetLastError();
        if (ib) cudaFreeAsync(ib, st);
        return fail(KNNG_E_NOMEM, "cannot allocate the batch graph");
    }
    std::vector<knng_iter_stats> hist;
    s = knng_build(vec_new, dt, n_new, d, k, metric, iters, sample_size, seed, static_cast<uint32_t*>(ib),
                   static_cast<float*>(db), nullptr, 0, stream);
    if (s == KNNG_OK) {
        hist = g_last_stats;
        s = knng_merge(vec_old, n_old, ids_old, dists_old, vec_new, n_new, static_cast<const uint32_t*>(ib),
                       static_cast<const float*>(db), dt, d, k, metric, merge_iters, sample_size, 0, seed, out_ids,
                       out_dists, nullptr, 0, stream);
        if (s == KNNG_OK) hist.insert(hist.end(), g_last_stats.begin(), g_last_stats.end());
    }
    cudaFreeAsync(ib, st);
    cudaFreeAsync(db, st);
    cudaStreamSynchronize(st);
    if (s == KNNG_OK) g_last_stats = hist;
    return s;
}

// ------------------------------------------------------------ multi-GPU
knng_status knng_get_unique_id(void* host_out128) {
    if (!host_out128) return fail(KNNG_E_USAGE, "null pointer argument");
    NcclApi& A = NcclApi::get();
    if (!A.ok()) return fail(KNNG_E_NCCL, "%s", A.error.c_str());
    ncclUniqueId id;
    const ncclResult_t r = A.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(KNNG_E_NCCL, "ncclGetUniqueId: %s", A.GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(host_out128, &id, sizeof(id));
    return KNNG_OK;
}

knng_status knng_comm_init(int32_t rank, int32_t world, const void* host_id128, void** comm) {
    if (!host_id128 || !comm) return fail(KNNG_E_USAGE, "null pointer argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(KNNG_E_USAGE, "rank must be in [0, world)");
    NcclApi& A = NcclApi::get();
    if (!A.ok()) return fail(KNNG_E_NCCL, "%s", A.error.c_str());
    ncclUniqueId id;
    memcpy(&id, host_id128, sizeof(id));
    auto* c = new NcclComm();
    c->rank = rank;
    c->world = world;
    const ncclResult_t r = A.CommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        delete c;
        return fail(KNNG_E_NCCL, "ncclCommInitRank: %s", A.GetErrorString(r));
    }
    *comm = static_cast<Comm*>(c);
    return KNNG_OK;
}

knng_status knng_comm_init_local(int32_t world, void** host_comms) {
    if (!host_comms || world < 1) return fail(KNNG_E_USAGE, "bad arguments");
    auto hub = std::make_shared<Hub>(world);
    for (int r = 0; r < world; ++r) {
        auto* c = new LocalComm();
        c->rank = r;
        c->world = world;
        c->hub = hub;
        host_comms[r] = static_cast<Comm*>(c);
    }
    return KNNG_OK;
}

knng_status knng_comm_destroy(void* comm) {
    delete static_cast<Comm*>(comm);
    return KNNG_OK;
}

knng_status knng_build_sharded(void* comm, const void* local_vectors, int64_t n_local, int64_t global_offset,
                               int64_t n_total, knng_dtype dt, int32_t d, int32_t k, knng_metric metric,
                               int32_t iters, int32_t merge_iters, const int32_t* host_level_iters,
                               int32_t sample_size, uint64_t seed, uint32_t* out_ids_local,
                               float* out_dists_local, void* stream) {
    if (!comm) return fail(KNNG_E_USAGE, "null communicator");
    Comm& C = *static_cast<Comm*>(comm);
    knng_status s = check_common(dt, n_local, d, k, metric, sample_size);
    if (s) return s;
    if (k > 32 && C.world > 1) return fail(KNNG_E_USAGE, "the GGM tree merges one-segment lists (k <= 32)");
    if (C.world & (C.world - 1)) return fail(KNNG_E_USAGE, "the world size must be a power of two");
    if (n_total != n_local * C.world) return fail(KNNG_E_USAGE, "n_total must be world * n_local (equal shards)");
    if (global_offset != static_cast<int64_t>(C.rank) * n_local)
        return fail(KNNG_E_USAGE, "global_offset must be rank * n_local");
    if (n_total >= 0xFFFFFFFFll) return fail(KNNG_E_USAGE, "n_total must be < 2^32 - 1");
    if (iters < 1 || iters > kMaxIters) return fail(KNNG_E_USAGE, "iters must be in [1, %d]", kMaxIters);
    int levels = 0;
    while ((1 << levels) < C.world) ++levels;
    for (int l = 0; l < levels; ++l) {
        const int mi = host_level_iters ? host_level_iters[l] : merge_iters;
        if (mi < 0 || mi > kMaxIters) return fail(KNNG_E_USAGE, "merge iterations must be in [0, %d]", kMaxIters);
    }
    if (!is_device_ptr(local_vectors) || !is_device_ptr(out_ids_local) || !is_device_ptr(out_dists_local))
        return fail(KNNG_E_USAGE, "vectors and outputs must be device pointers");
    return run_sharded(C, local_vectors, n_local, global_offset, n_total, dt, d, k, metric, iters, merge_iters,
                       host_level_iters, sample_size, seed, out_ids_local, out_dists_local,
                       static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------ introspection
int32_t knng_last_stats(knng_iter_stats* host_out, int32_t max_iters) {
    const int32_t m = static_cast<int32_t>(g_last_stats.size()) < max_iters ? static_cast<int32_t>(g_last_stats.size()) : max_iters;
    for (int32_t i = 0; i < m; ++i) host_out[i] = g_last_stats[i];
    return m;
}

int64_t knng_launch_count(void) { return g_launches.load(); }

void knng_set_timing(int32_t enable) { g_timing.store(enable ? 1 : 0); }

void knng_reset_timing(void) {
    std::lock_guard<std::mutex> lk(g_time_mu);
    g_times.clear();
}

int32_t knng_kernel_time(const char* name, double* total_ms, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_time_mu);
    auto it = g_times.find(name ? name : "");
    if (it == g_times.end()) {
        if (total_ms) *total_ms = 0.0;
        if (launches) *launches = 0;
        return 0;
    }
    if (total_ms) *total_ms = it->second.first;
    if (launches) *launches = it->second.second;
    return 1;
}

const char* knng_last_error(void) { return g_err.c_str(); }

const char* knng_status_string(knng_status s) {
    switch (s) {
        case KNNG_OK: return "KNNG_OK";
        case KNNG_E_USAGE: return "KNNG_E_USAGE";
        case KNNG_E_DOMAIN: return "KNNG_E_DOMAIN";
        case KNNG_E_NOMEM: return "KNNG_E_NOMEM";
        case KNNG_E_CUDA: return "KNNG_E_CUDA";
        case KNNG_E_NCCL: return "KNNG_E_NCCL";
        case KNNG_E_INTERNAL: return "KNNG_E_INTERNAL";
    }
    return "unknown";
}

knng_status knng_set_option(const char* name, int64_t value) {
    if (!name) return fail(KNNG_E_USAGE, "null option name");
    if (strcmp(name, "exact_u8") == 0) {
        g_opt_exact_u8.store(value ? 1 : 0);
        return KNNG_OK;
    }
    if (strcmp(name, "update") == 0) {
        if (value < 0 || value > 3) return fail(KNNG_E_USAGE, "update must be in [0, 3]");
        g_opt_update.store(static_cast<int>(value));
        return KNNG_OK;
    }
#ifdef KNNG_WS_PROF
    if (strcmp(name, "ws_probe") == 0) {  // profiling build only
        const int v = static_cast<int>(value);
        cudaMemcpyToSymbol(g_ws_probe, &v, sizeof(int));
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(g_ws_prof, z, sizeof(z));
        return KNNG_OK;
    }
#endif
    if (strcmp(name, "join_kernel") == 0) {
        if (value < 0 || value > 4) return fail(KNNG_E_USAGE, "join_kernel must be 0..4");
        g_opt_join_kernel.store(static_cast<int>(value));
        return KNNG_OK;
    }
    return fail(KNNG_E_USAGE, "unknown or read-only option '%s'", name);
}

knng_status knng_get_option(const char* name, int64_t* host_value) {
    if (!name || !host_value) return fail(KNNG_E_USAGE, "null argument");
    if (strcmp(name, "exact_u8") == 0) *host_value = g_opt_exact_u8.load();
    else if (strcmp(name, "join_kernel") == 0) *host_value = g_opt_join_kernel.load();
    else if (strcmp(name, "update") == 0) *host_value = g_opt_update.load();
    else if (strcmp(name, "last_exact_u8") == 0) *host_value = g_last_exact_u8;
#ifdef KNNG_WS_PROF
    else if (strncmp(name, "ws_prof", 7) == 0) {  // profiling build only
        unsigned long long v[32];
        cudaMemcpyFromSymbol(v, g_ws_prof, sizeof(v));
        *host_value = static_cast<int64_t>(v[atoi(name + 7)]);
    }
#endif
    else return fail(KNNG_E_USAGE, "unknown option '%s'", name);
    return KNNG_OK;
}

int32_t knng_abi_version(void) { return 2; }

}  // extern "C"

// the out-of-memory all-pairs construction: host orchestration
#include "ooc_api.cuh"
