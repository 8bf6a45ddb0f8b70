// libaddkern_b200: plan-time geometry, operator apply, FFT stage and the C ABI.
//
// Canonical grid layout (all entry points): windows ordered by decreasing
// window length q (stable), window w's R grids consecutive:
//   grid(w, r) = grids + R * canon_off[w] + r * n^q[w]
// so that all windows of one length form one contiguous cuFFT batch.
#include <cub/cub.cuh>
#include <cufft.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "ak_common.cuh"
#include "ak_kernels.cuh"
#include "ak_q3w.cuh"
#include "ak_q3m.cuh"
#include "ak_q3c.cuh"
#include "ak_q2c.cuh"
#include "ak_q3r.cuh"
#include "ak_q1r.cuh"
#include "ak_q2r.cuh"
#include "ak_fft3.cuh"
#include "ak_q3b.cuh"
#include "ak_q3h.cuh"

using namespace ak;

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define AK_CUDA(call)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(e_ == cudaErrorMemoryAllocation ? AK_ERR_ALLOC : AK_ERR_CUDA,       \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                \
    } while (0)

#define AK_CUFFT(call)                                                                      \
    do {                                                                                    \
        cufftResult r_ = (call);                                                            \
        if (r_ != CUFFT_SUCCESS)                                                            \
            return fail(AK_ERR_CUFFT, std::string(#call) + ": cufft error " + std::to_string((int)r_)); \
    } while (0)

#define AK_TRY(call)              \
    do {                          \
        int rc_ = (call);         \
        if (rc_ != AK_OK) return rc_; \
    } while (0)

int ak_internal_fail(int code, const char* msg) { return fail(code, msg); }
void ak_internal_count(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static int launched() {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(AK_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    return AK_OK;
}

// ---------------------------------------------------------------------------
// per-kernel device timing (ak_prof_*): off by default; when on, each launch site
// brackets its kernel with two CUDA events on the launching stream.

static std::atomic<bool> g_prof_on{false};
static std::mutex g_prof_mu;
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof;

struct ProfScope {
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    explicit ProfScope(cudaStream_t s) : st(s) {
        if (g_prof_on.load(std::memory_order_relaxed) && cudaEventCreate(&a) == cudaSuccess) cudaEventRecord(a, st);
    }
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;
    // after the launch: error check + launch count, then the closing event
    int done(const char* name, bool counted = false) {
        const int rc = counted ? AK_OK : launched();
        close(name);
        return rc;
    }
    void close(const char* name) {
        if (!a) return;
        cudaEvent_t b = nullptr;
        if (cudaEventCreate(&b) == cudaSuccess && cudaEventRecord(b, st) == cudaSuccess) {
            std::lock_guard<std::mutex> lk(g_prof_mu);
            g_prof.push_back(ProfRec{name, a, b});
            a = nullptr;
        } else if (b) {
            cudaEventDestroy(b);
        }
    }
    ~ProfScope() {
        if (a) cudaEventDestroy(a);
    }
};

static void prof_clear_locked() {
    for (auto& r : g_prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.clear();
}

extern "C" int ak_prof_enable(int32_t on) {
    g_prof_on.store(on != 0);
    return AK_OK;
}

extern "C" int ak_prof_reset(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof.empty()) cudaDeviceSynchronize();
    prof_clear_locked();
    return AK_OK;
}

extern "C" int64_t ak_prof_report(char* buf, int64_t cap) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof.empty() && cudaDeviceSynchronize() != cudaSuccess) return fail(AK_ERR_CUDA, "device synchronize failed");
    std::vector<std::string> names;
    std::map<std::string, std::pair<int64_t, double>> agg;
    for (auto& r : g_prof) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
        auto it = agg.find(r.name);
        if (it == agg.end()) {
            names.push_back(r.name);
            agg[r.name] = {1, (double)ms};
        } else {
            it->second.first += 1;
            it->second.second += ms;
        }
    }
    std::string out;
    for (auto& nm : names) {
        char line[256];
        snprintf(line, sizeof line, "%s\t%lld\t%.6f\n", nm.c_str(), (long long)agg[nm].first, agg[nm].second);
        out += line;
    }
    if (buf && cap > 0) {
        const int64_t k = std::min<int64_t>(cap - 1, (int64_t)out.size());
        memcpy(buf, out.data(), (size_t)k);
        buf[k] = 0;
    }
    return (int64_t)out.size() + 1;
}

// ---------------------------------------------------------------------------
// device allocations of the library's own buffers.  Checked builds (-DAK_CHECKED,
// tools/checked_build.py) surround each with guard bands that are verified after
// every entry point, and poison the buffer with NaN bytes so that a read of memory
// no kernel wrote shows up in the results (a memcheck / initcheck substitute).

#ifdef AK_CHECKED
static constexpr size_t kGuard = 4096;
struct GuardRec {
    char* base;
    size_t bytes;
    std::string name;
};
static std::mutex g_guard_mu;
static std::map<void*, GuardRec> g_guards;

static cudaError_t ak_malloc_named(void** p, size_t bytes, const char* name) {
    char* base = nullptr;
    cudaError_t e = cudaMalloc(&base, bytes + 2 * kGuard);
    if (e != cudaSuccess) {
        *p = nullptr;
        return e;
    }
    cudaMemset(base, 0xA5, kGuard);
    cudaMemset(base + kGuard + bytes, 0xA5, kGuard);
    cudaMemset(base + kGuard, 0xFF, bytes);
    *p = base + kGuard;
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guards[*p] = GuardRec{base, bytes, name};
    return cudaSuccess;
}

static void ak_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_guard_mu);
    auto it = g_guards.find(p);
    if (it != g_guards.end()) {
        cudaFree(it->second.base);
        g_guards.erase(it);
    } else {
        cudaFree(p);
    }
}

static int fail(int code, const std::string& msg);
static int guards_verify(const char* where) {
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(AK_ERR_CUDA, std::string("device fault in ") + where);
    std::lock_guard<std::mutex> lk(g_guard_mu);
    std::vector<unsigned char> h(2 * kGuard);
    for (auto& kv : g_guards) {
        const GuardRec& r = kv.second;
        cudaMemcpy(h.data(), r.base, kGuard, cudaMemcpyDeviceToHost);
        cudaMemcpy(h.data() + kGuard, r.base + kGuard + r.bytes, kGuard, cudaMemcpyDeviceToHost);
        for (unsigned char c : h)
            if (c != 0xA5) return fail(AK_ERR_CUDA, "guard band of " + r.name + " overwritten (" + where + ")");
    }
    return AK_OK;
}
#else
static inline cudaError_t ak_malloc_named(void** p, size_t bytes, const char*) { return cudaMalloc(p, bytes); }
static inline void ak_free(void* p) { cudaFree(p); }
static inline int guards_verify(const char*) { return AK_OK; }
#endif
#define AK_MALLOC(ptr, bytes) ak_malloc_named(reinterpret_cast<void**>(ptr), (bytes), #ptr)

static inline int64_t ipow_rt(int64_t b, int q) {
    int64_t r = 1;
    for (int i = 0; i < q; ++i) r *= b;
    return r;
}

// ---------------------------------------------------------------------------
// geometry

struct ak_geom {
    int n = 0, P = 0;
    int64_t N = 0;
    std::vector<int> q;                 // per window
    std::vector<int64_t> canon_off;     // per window (R = 1 units)
    int64_t canon_total = 0;            // sum n^q
    int64_t* canon_off_d = nullptr;
    ak_window_fn wf{};
    Point* pts = nullptr;               // [P][N]
    std::vector<int64_t> rows_in;       // per window: rows it uses (N, or the mask count; sorted first)
    WorkItem* items = nullptr;
    int64_t nitems = 0;
    int64_t item_begin[4] = {0, 0, 0, 0}, item_end[4] = {0, 0, 0, 0};
    std::vector<int> windows_of_q[4];   // window ids per q, canonical order
    int sedge[4] = {0, 16, 8, 4};       // supercell edge (cells) per q (must match SuperCell<q>)
    int sedge_i3 = 4;                   // supercell edge of the 3-D interpolation items
    bool trim3 = false;                 // 12-tap table whose outer tap pair is zero (a padded 10-tap window)
    int chunk[4] = {0, 2048, 1024, 2048};  // maximum points per work item, per q
    int64_t iitem_begin3 = 0, iitem_end3 = 0;  // 3-D interpolation items (== spread items unless split)
    // cached 3-D window weights (plan-time table, see ak_q3w.cuh)
    bool cached = false;
    ak_tuning tune{};                   // plan-time kernel selection (ak_geom_create_ex)
    std::string desc;                   // ak_geom_describe
    double* W3 = nullptr;               // [P3][N][3T]
    CellIdx* CI3 = nullptr;             // [P3][N]
    bool cached2 = false;               // 2-D weight table present (ak_q2c.cuh kernels)
    double* W2 = nullptr;               // [P2][N][2T]
    CellIdx* CI2 = nullptr;             // [P2][N]
    int64_t* wshift_d = nullptr;        // per window: (w - rank_q(w)) * N, rank among windows of its q
    // Occupied box of each 3-D window's grid: per axis the cyclic index range [lo, lo + L)
    // (mod n) that holds every footprint of the window's points, L a multiple of 16
    // (full axis: lo = 0, L = n).  The fused transforms skip the rest (zero on the way in,
    // never read on the way out).  [P][lo0, L0, lo1, L1, lo2, L2].
    std::vector<int> box;
    int* box_d = nullptr;
};

extern "C" void ak_tuning_default(ak_tuning* t) {
    if (!t) return;
    t->weight_tables = 1;
    t->cell_items3 = 0;
    t->dense_cells3 = 300.0;       // measured on B200, config-4 data at 125k..2M points
    t->dense_cells3_interp = 64.0;
    t->cell_items2 = 0;
    t->dense_cells2 = 2.0;         // config 2 at ~5 points per cell: 2.6x faster with single-cell items
    t->chunk3 = 0;
    t->rhs_pair_spread = 1;
    t->fused_fft3 = 1;
    t->generic_kernels = 0;
    t->sparse_warps = 2;
    t->tc_spread3 = 3;
}

__global__ void k_count_nonzero(const int* __restrict__ counts, int total, int* __restrict__ nz) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool on = i < total && counts[i] > 0;
    const unsigned b = __ballot_sync(0xffffffffu, on);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(nz, __popc(b));
}

// Maximum points per work item.  Items are processed one per CTA in largest-first
// order, so the largest item bounds the tail: the cap is half the average work per
// resident CTA slot (SMs x 8), within [64, 2048] (q = 3) / [64, 1024] (q = 2);
// 2048 for q = 1.  Measured on clustered config-4 data at 30k nodes: the fixed 2048
// cap left a few 800-point supercell items as the tail (spread 0.140 -> 0.097 ms,
// interp 0.157 -> 0.082 ms with the adaptive cap).  ak_tuning::chunk3 pins q = 3.
static int chunk_for(int q, int64_t point_windows, const ak_tuning& t) {
    if (q == 1) return 2048;
    if (q == 3 && t.chunk3 >= 64 && t.chunk3 <= 65536) return t.chunk3;
    static int slots = 0;
    if (!slots) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        slots = std::max(1, sms) * 8;
    }
    const int64_t hi = q == 3 ? 2048 : 1024;
    return (int)std::max<int64_t>(64, std::min<int64_t>(hi, point_windows / (2 * (int64_t)slots)));
}

// mask (optional, the window's N-row slice): rows with mask 0 get the key `sentinel`,
// which sorts after every cell key, and stay out of the histogram (no work item
// covers them: a row-subset window for cell-slab sharding).
__global__ void k_keys(const double* __restrict__ X, int64_t ld, int q, int c0, int c1, int c2, int n, int S,
                       int nsc, int64_t N, uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                       int* __restrict__ counts, int* __restrict__ bad, const uint8_t* __restrict__ mask = nullptr,
                       uint32_t sentinel = 0)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int col[3] = {c0, c1, c2};
    const bool in = !mask || mask[i];
    int sc = 0, sub = 0;
    for (int a = 0; a < q; ++a) {
        double x = X[i * ld + col[a]];
        if (!(x >= -0.5 && x < 0.5)) {
            atomicOr(bad, 1);
            x = 0.0;
        }
        const double t = (x + 0.5) * n;
        int c = (int)floor(t);
        if (c >= n) c -= n;
        sc = sc * nsc + c / S;
        sub = sub * S + c % S;
    }
    int sq = 1;
    for (int a = 0; a < q; ++a) sq *= S;
    keys[i] = in ? (uint32_t)sc * (uint32_t)sq + (uint32_t)sub : sentinel;
    vals[i] = (int32_t)i;
    if (!in) return;
    // warp-aggregated histogram update (clustered data puts many lanes in one supercell)
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, sc);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&counts[sc], __popc(peers));
}

__global__ void k_points(const double* __restrict__ X, int64_t ld, int q, int c0, int c1, int c2, int n,
                         const int32_t* __restrict__ order, int64_t N, Point* __restrict__ out)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const int i = order[j];
    const int col[3] = {c0, c1, c2};
    Point p;
    p.s[0] = p.s[1] = p.s[2] = 0.0;
    int packed = 0;
    for (int a = 0; a < q; ++a) {
        double x = X[(int64_t)i * ld + col[a]];
        if (!(x >= -0.5 && x < 0.5)) x = 0.0;
        const double t = (x + 0.5) * n;
        const double fl = floor(t);
        const double frac = t - fl;            // exact
        int c = (int)fl;
        if (c >= n) c -= n;
        p.s[a] = fma(2.0, frac, -1.0);
        packed |= c << (10 * a);
    }
    p.cell = packed;
    p.idx = i;
    out[j] = p;
}

__global__ void k_items(const int* __restrict__ counts, const int* __restrict__ starts, int nsc_total, int q,
                        int nsc, int chunk, int64_t pt_base, int w, int* __restrict__ counter,
                        WorkItem* __restrict__ items)
{
    const int sc = blockIdx.x * blockDim.x + threadIdx.x;
    if (sc >= nsc_total) return;
    const int cnt = counts[sc];
    if (cnt == 0) return;
    const int k = (cnt + chunk - 1) / chunk;
    const int size = (cnt + k - 1) / k;
    const int base = atomicAdd(counter, k);
    int s[3] = {0, 0, 0};
    int rest = sc;
    for (int a = q - 1; a >= 0; --a) {
        s[a] = rest % nsc;
        rest /= nsc;
    }
    const int packed = s[0] | (s[1] << 10) | (s[2] << 20);
    for (int j = 0; j < k; ++j) {
        WorkItem it;
        it.window = w;
        it.sc = packed;
        it.start = (int)(pt_base + starts[sc] + (int64_t)j * size);
        it.count = min(size, cnt - j * size);
        items[base + j] = it;
    }
}

// Run boundaries of the sorted keys: a key's run is [kstart, kend) (0/0 when absent).
__global__ void k_key_bounds(const uint32_t* __restrict__ keys, int64_t N, int* __restrict__ kstart,
                             int* __restrict__ kend, int64_t nkeys)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t k = keys[i];
    if ((int64_t)k >= nkeys) return;   // masked-out rows (sentinel key)
    if (i == 0 || keys[i - 1] != k) kstart[k] = (int)i;
    if (i == N - 1 || keys[i + 1] != k) kend[k] = (int)(i + 1);
}

// Single-cell work items (3-D) from the run of each key of a (supercell, cell) sort:
// key = supercell * S^3 + (u0 * S + u1) * S + u2, cell = supercell digit * S + u.
__global__ void k_items_cells(const int* __restrict__ kstart, const int* __restrict__ kend, int64_t nkeys, int S,
                              int nsc, int chunk, int64_t pt_base, int w, int* __restrict__ counter,
                              WorkItem* __restrict__ items)
{
    const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (key >= nkeys) return;
    const int cnt = kend[key] - kstart[key];
    if (cnt <= 0) return;
    const int S3 = S * S * S;
    const int sc = (int)(key / S3), sub = (int)(key - (int64_t)sc * S3);
    const int s0 = sc / (nsc * nsc), s1 = (sc / nsc) % nsc, s2 = sc % nsc;
    const int u0 = sub / (S * S), u1 = (sub / S) % S, u2 = sub % S;
    const int packed = (s0 * S + u0) | ((s1 * S + u1) << 10) | ((s2 * S + u2) << 20);
    const int k = (cnt + chunk - 1) / chunk;
    const int size = (cnt + k - 1) / k;
    const int base = atomicAdd(counter, k);
    for (int j = 0; j < k; ++j) {
        WorkItem it;
        it.window = w;
        it.sc = packed;
        it.start = (int)(pt_base + kstart[key] + (int64_t)j * size);
        it.count = min(size, cnt - j * size);
        items[base + j] = it;
    }
}

extern "C" const char* ak_last_error(void) { return g_err.c_str(); }
extern "C" const char* ak_version(void) { return "addkern_b200 0.1.0 (sm_100a)"; }
extern "C" int64_t ak_launch_count(void) { return g_launches.load(); }

extern "C" int ak_geom_destroy(ak_geom* g) {
    if (!g) return AK_OK;
    ak_free(g->pts);
    ak_free(g->items);
    ak_free(g->canon_off_d);
    ak_free(g->W3);
    ak_free(g->CI3);
    ak_free(g->W2);
    ak_free(g->CI2);
    ak_free(g->wshift_d);
    ak_free(g->box_d);
    delete g;
    return AK_OK;
}

// Occupied boxes of the 3-D windows (ak_geom::box) from the spread work items: a cell c
// of a T-tap window touches grid indices c - (T/2 - 1) .. c + T/2 (mod n); per axis the
// box is the complement of the longest cyclic run of untouched indices, rounded up to a
// multiple of 16 (the fused transforms' GEMM tiling).
static void geom_boxes(ak_geom* g, const std::vector<WorkItem>& items, int64_t ib, int64_t ie) {
    const int n = g->n, P = g->P, T = g->wf.taps, S = g->sedge[3];
    g->box.assign((size_t)P * 6, 0);
    std::vector<std::vector<char>> occ((size_t)P * 3, std::vector<char>(n, 0));
    for (int64_t i = ib; i < ie; ++i) {
        const WorkItem& it = items[(size_t)i];
        for (int a = 0; a < 3; ++a) {
            const int c = ((it.sc >> (10 * a)) & 1023) * S;
            for (int k = 0; k < S && c + k < n; ++k) occ[(size_t)it.window * 3 + a][c + k] = 1;
        }
    }
    for (int w = 0; w < P; ++w)
        for (int a = 0; a < 3; ++a) {
            int lo = 0, L = n;
            if (g->q[w] == 3 && n % 16 == 0) {
                std::vector<char> touched(n, 0);
                const auto& o = occ[(size_t)w * 3 + a];
                for (int c = 0; c < n; ++c)
                    if (o[c])
                        for (int t = 0; t < T; ++t) touched[((c - (T / 2 - 1) + t) % n + n) % n] = 1;
                // longest cyclic run of untouched indices
                int best = 0, best_end = 0, run = 0;
                for (int i = 0; i < 2 * n; ++i) {
                    run = touched[i % n] ? 0 : std::min(run + 1, n);
                    if (run > best) {
                        best = run;
                        best_end = i % n;
                    }
                }
                if (best == n) {
                    L = 16;   // no points: any small box
                } else if (best > 0) {
                    lo = (best_end + 1) % n;
                    L = n - best;
                }
                L = (L + 15) / 16 * 16;
                if (L >= n) {
                    lo = 0;
                    L = n;
                }
            }
            g->box[(size_t)w * 6 + 2 * a] = lo;
            g->box[(size_t)w * 6 + 2 * a + 1] = L;
        }
}

// Mean points per occupied cell of window w (bins at S = 1); -1 when the probe fails.
static double mean_occupancy(const double* X, int64_t ld, const int32_t* cols, int w, int q, int n, int64_t N,
                             cudaStream_t st, const uint8_t* mask = nullptr, int64_t n_in = -1)
{
    const int tot = (int)ipow_rt(n, q);
    int *cnt = nullptr, *aux = nullptr;
    uint32_t* kk = nullptr;
    int32_t* vv = nullptr;
    double mean = -1.0;
    if (cudaMalloc(&cnt, sizeof(int) * tot) == cudaSuccess && cudaMalloc(&aux, sizeof(int) * 2) == cudaSuccess &&
        cudaMalloc(&kk, sizeof(uint32_t) * N) == cudaSuccess && cudaMalloc(&vv, sizeof(int32_t) * N) == cudaSuccess) {
        cudaMemsetAsync(cnt, 0, sizeof(int) * tot, st);
        cudaMemsetAsync(aux, 0, sizeof(int) * 2, st);
        k_keys<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(X, ld, q, cols[3 * w], cols[3 * w + 1], cols[3 * w + 2],
                                                             n, 1, n, N, kk, vv, cnt, aux, mask, 0u);
        k_count_nonzero<<<(tot + 255) / 256, 256, 0, st>>>(cnt, tot, aux + 1);
        g_launches.fetch_add(2);
        int h[2] = {0, 0};
        if (cudaMemcpyAsync(h, aux, sizeof(h), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
            cudaStreamSynchronize(st) == cudaSuccess && h[1] > 0)
            mean = (double)(n_in >= 0 ? n_in : N) / h[1];
    }
    cudaGetLastError();
    cudaFree(cnt);
    cudaFree(aux);
    cudaFree(kk);
    cudaFree(vv);
    return mean;
}

// Device scratch released when it goes out of scope (every return path of geom_build).
struct Scratch {
    std::vector<void*> bufs;
    ~Scratch() {
        for (void* b : bufs) ak_free(b);
    }
    template <typename T>
    cudaError_t alloc(T** p, size_t bytes) {
        *p = nullptr;
        const cudaError_t e = AK_MALLOC(p, bytes);
        if (e == cudaSuccess) bufs.push_back(*p);
        return e;
    }
};

// masks: optional device uint8 [P][N] (row r belongs to window w iff masks[w N + r]);
// n_in: host per-window row counts of the masks (occupancy probes)
static int geom_build(ak_geom* g, const int32_t* cols, const double* X, int64_t ld, cudaStream_t st,
                      const uint8_t* masks = nullptr, const int64_t* n_in = nullptr) {
    auto wmask = [&](int w) { return masks ? masks + (int64_t)w * g->N : nullptr; };
    auto win_rows = [&](int w) { return n_in ? n_in[w] : (int64_t)-1; };
    const int n = g->n, P = g->P;
    const int64_t N = g->N;
    // canonical order: q descending, stable
    int64_t off = 0;
    g->canon_off.assign(P, 0);
    for (int q = 3; q >= 1; --q)
        for (int w = 0; w < P; ++w)
            if (g->q[w] == q) {
                g->canon_off[w] = off;
                off += ipow_rt(n, q);
                g->windows_of_q[q].push_back(w);
            }
    g->canon_total = off;
    AK_CUDA(AK_MALLOC(&g->canon_off_d, sizeof(int64_t) * P));
    AK_CUDA(cudaMemcpyAsync(g->canon_off_d, g->canon_off.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, st));

    AK_CUDA(AK_MALLOC(&g->pts, sizeof(Point) * (size_t)std::max<int64_t>(1, N * P)));
    int max_nsc_total = 1;
    bool cached = g->wf.taps == 12 && N > 0 && g->tune.weight_tables;
    if (cached) {
        // plan-time weight tables (filled once the points are sorted, below)
        const int64_t P3 = (int64_t)g->windows_of_q[3].size(), P2 = (int64_t)g->windows_of_q[2].size();
        const int T = g->wf.taps;
        bool ok = AK_MALLOC(&g->wshift_d, sizeof(int64_t) * P) == cudaSuccess;
        if (ok && P3 > 0)
            ok = AK_MALLOC(&g->W3, sizeof(double) * P3 * N * 3 * T) == cudaSuccess &&
                 AK_MALLOC(&g->CI3, sizeof(CellIdx) * P3 * N) == cudaSuccess;
        if (ok && P2 > 0)
            ok = AK_MALLOC(&g->W2, sizeof(double) * P2 * N * 2 * T) == cudaSuccess &&
                 AK_MALLOC(&g->CI2, sizeof(CellIdx) * P2 * N) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();  // not enough memory for the tables: evaluate weights per pass
            ak_free(g->W3);
            ak_free(g->CI3);
            ak_free(g->W2);
            ak_free(g->CI2);
            ak_free(g->wshift_d);
            g->W3 = g->W2 = nullptr;
            g->CI3 = g->CI2 = nullptr;
            g->wshift_d = nullptr;
            cached = false;
        }
    }
    // Supercell edges.  3-D windows: the spread and the interpolation may use different
    // work items over the same sorted points: single-cell items pay off for the
    // interpolation from ~64 points per occupied cell, for the spread only from ~300
    // (below that its per-cell register flush costs more than the supercell tile;
    // config-4 data: 210 points per cell at 500k nodes, 427 at 1M).
    int s3 = (g->tune.cell_items3 == 1 || g->tune.cell_items3 == 2) ? g->tune.cell_items3 : 0;
    if (s3 == 1 && !cached) s3 = 2;  // single-cell kernels exist for the cached-weight path only
    int si3 = s3;
    if (s3 == 0) {
        s3 = si3 = 2;
        // (the probe and the split item lists keep one int per cell: only for grids up to 256^3)
        if (cached && !g->windows_of_q[3].empty() && n <= 256) {
            const int w0 = g->windows_of_q[3][0];
            const double occ = mean_occupancy(X, ld, cols, w0, 3, n, N, st, wmask(w0), win_rows(w0));
            if (occ >= g->tune.dense_cells3) s3 = 1;
            if (occ >= g->tune.dense_cells3_interp) si3 = 1;
        }
    }
    if (s3 == 1) si3 = 1;
    if (n > 256) si3 = s3;  // no split item lists for huge grids (see above)
    const bool split3 = (si3 == 1 && s3 != 1);
    int s2 = (g->tune.cell_items2 == 1 || g->tune.cell_items2 == 8) ? g->tune.cell_items2 : 0;
    if (s2 == 1 && !cached) s2 = 8;
    if (s2 == 0) {
        s2 = 8;
        if (cached && !g->windows_of_q[2].empty() && n <= 4096 &&
            mean_occupancy(X, ld, cols, g->windows_of_q[2][0], 2, n, N, st, wmask(g->windows_of_q[2][0]),
                           win_rows(g->windows_of_q[2][0])) >= g->tune.dense_cells2)
            s2 = 1;
    }
    g->sedge[2] = s2;
    g->sedge[3] = s3;
    g->sedge_i3 = si3;
    for (int q = 1; q <= 3; ++q) {
        int64_t pw = 0;   // point-windows of this length (masked rows excluded)
        for (int w : g->windows_of_q[q]) pw += n_in ? n_in[w] : N;
        g->chunk[q] = chunk_for(q, pw, g->tune);
    }
    int64_t tcap = 1;     // per-window item capacity of the staging buffer
    int64_t keyspace = 1; // 3-D sort-key space (cells in supercell order) when split
    for (int w = 0; w < P; ++w) {
        const int S = g->sedge[g->q[w]];
        const int nsc = (n + S - 1) / S;
        const int tot = (int)ipow_rt(nsc, g->q[w]);
        max_nsc_total = std::max(max_nsc_total, tot);
        const int ch = g->chunk[g->q[w]];
        tcap = std::max<int64_t>(tcap, (N + ch - 1) / ch + tot);
        if (g->q[w] == 3 && split3) {
            keyspace = std::max<int64_t>(keyspace, (int64_t)tot * S * S * S);
            tcap = std::max<int64_t>(tcap, (N + ch - 1) / ch + std::min<int64_t>(N, (int64_t)tot * S * S * S));
        }
    }

    Scratch scratch;  // plan-time buffers, released on every return path
    uint32_t *keys = nullptr, *keys2 = nullptr;
    int32_t *vals = nullptr, *vals2 = nullptr;
    int *counts = nullptr, *starts = nullptr, *dflags = nullptr, *kstart = nullptr, *kend = nullptr;
    WorkItem* titems = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0, need = 0;
    const int64_t NN = std::max<int64_t>(N, 1);
    AK_CUDA(scratch.alloc(&keys, sizeof(uint32_t) * NN));
    AK_CUDA(scratch.alloc(&keys2, sizeof(uint32_t) * NN));
    AK_CUDA(scratch.alloc(&vals, sizeof(int32_t) * NN));
    AK_CUDA(scratch.alloc(&vals2, sizeof(int32_t) * NN));
    AK_CUDA(scratch.alloc(&counts, sizeof(int) * max_nsc_total));
    AK_CUDA(scratch.alloc(&starts, sizeof(int) * max_nsc_total));
    AK_CUDA(scratch.alloc(&dflags, sizeof(int) * 2));  // [0] bad, [1] item counter
    AK_CUDA(scratch.alloc(&titems, sizeof(WorkItem) * tcap));
    if (split3) {
        AK_CUDA(scratch.alloc(&kstart, sizeof(int) * keyspace));
        AK_CUDA(scratch.alloc(&kend, sizeof(int) * keyspace));
    }
    AK_CUDA(cudaMemsetAsync(dflags, 0, sizeof(int) * 2, st));
    cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys2, vals, vals2, (int)N, 0, 32, st);
    temp_bytes = need;
    cub::DeviceScan::ExclusiveSum(nullptr, need, counts, starts, max_nsc_total, st);
    temp_bytes = std::max(temp_bytes, need);
    AK_CUDA(scratch.alloc(&temp, std::max<size_t>(temp_bytes, 16)));

    int rc = AK_OK;
    std::vector<WorkItem> all;  // final order: q=3 spread | q=3 interp (split) | q=2 | q=1
    // staged items of one window -> host (the counter is reset per window)
    auto take = [&](std::vector<WorkItem>& dst) -> int {
        int cnt = 0;
        if (cudaMemcpyAsync(&cnt, dflags + 1, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(AK_ERR_CUDA, "item count read failed");
        const size_t at = dst.size();
        dst.resize(at + (size_t)cnt);
        if (cnt > 0 && (cudaMemcpyAsync(dst.data() + at, titems, sizeof(WorkItem) * cnt, cudaMemcpyDeviceToHost, st) !=
                            cudaSuccess ||
                        cudaStreamSynchronize(st) != cudaSuccess))
            return fail(AK_ERR_CUDA, "item copy failed");
        if (cudaMemsetAsync(dflags + 1, 0, sizeof(int), st) != cudaSuccess) return fail(AK_ERR_CUDA, "memset failed");
        return AK_OK;
    };
    // Largest items first (blocks are dispatched in index order: LPT-like tail).
    auto append_sorted = [&](std::vector<WorkItem>& v, int64_t& begin, int64_t& end) {
        if (v.size() > 1)
            std::stable_sort(v.begin(), v.end(), [](const WorkItem& a, const WorkItem& b) {
                if (a.count != b.count) return a.count > b.count;
                return a.start < b.start;
            });
        begin = (int64_t)all.size();
        all.insert(all.end(), v.begin(), v.end());
        end = (int64_t)all.size();
    };
    for (int q = 3; q >= 1 && rc == AK_OK; --q) {
        std::vector<WorkItem> spread_items, cell_items;
        for (int w : g->windows_of_q[q]) {
            const int S = g->sedge[q];
            const int nsc = (n + S - 1) / S;
            const int tot = (int)ipow_rt(nsc, q);
            int bits = 1;
            while ((int64_t)1 << bits < (int64_t)tot * ipow_rt(S, q)) ++bits;
            // masked rows: sentinel key 2^bits sorts after every cell (one more key bit)
            const uint32_t sentinel = (uint32_t)1 << bits;
            if (masks) ++bits;
            const int c0 = cols[3 * w], c1 = cols[3 * w + 1], c2 = cols[3 * w + 2];
            if (N == 0) continue;
            cudaMemsetAsync(counts, 0, sizeof(int) * tot, st);
            const int tb = 256;
            const int nblk = (int)((N + tb - 1) / tb);
            k_keys<<<nblk, tb, 0, st>>>(X, ld, q, c0, c1, c2, n, S, nsc, N, keys, vals, counts, dflags, wmask(w),
                                        sentinel);
            if ((rc = launched()) != AK_OK) break;
            size_t tb2 = temp_bytes;
            if (cub::DeviceRadixSort::SortPairs(temp, tb2, keys, keys2, vals, vals2, (int)N, 0, bits, st) != cudaSuccess) {
                rc = fail(AK_ERR_CUDA, "radix sort failed");
                break;
            }
            g_launches.fetch_add(1);
            k_points<<<nblk, tb, 0, st>>>(X, ld, q, c0, c1, c2, n, vals2, N, g->pts + (int64_t)w * N);
            if ((rc = launched()) != AK_OK) break;
            tb2 = temp_bytes;
            if (cub::DeviceScan::ExclusiveSum(temp, tb2, counts, starts, tot, st) != cudaSuccess) {
                rc = fail(AK_ERR_CUDA, "scan failed");
                break;
            }
            g_launches.fetch_add(1);
            k_items<<<(tot + 255) / 256, 256, 0, st>>>(counts, starts, tot, q, nsc, g->chunk[q], (int64_t)w * N, w,
                                                       dflags + 1, titems);
            if ((rc = launched()) != AK_OK || (rc = take(spread_items)) != AK_OK) break;
            if (q == 3 && split3) {
                // single-cell items over the same (supercell, cell)-sorted points: each cell is
                // one run of equal keys
                const int64_t nk = (int64_t)tot * S * S * S;
                cudaMemsetAsync(kstart, 0, sizeof(int) * nk, st);
                cudaMemsetAsync(kend, 0, sizeof(int) * nk, st);
                k_key_bounds<<<nblk, tb, 0, st>>>(keys2, N, kstart, kend, nk);
                if ((rc = launched()) != AK_OK) break;
                k_items_cells<<<(unsigned)((nk + 255) / 256), 256, 0, st>>>(kstart, kend, nk, S, nsc, g->chunk[3],
                                                                            (int64_t)w * N, w, dflags + 1, titems);
                if ((rc = launched()) != AK_OK || (rc = take(cell_items)) != AK_OK) break;
            }
        }
        if (rc != AK_OK) break;
        int bad = 0;
        if (cudaMemcpyAsync(&bad, dflags, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            rc = fail(AK_ERR_CUDA, "geometry sync failed");
            break;
        }
        if (bad) {
            rc = fail(AK_ERR_DOMAIN, "points must lie in [-1/2, 1/2)");
            break;
        }
        append_sorted(spread_items, g->item_begin[q], g->item_end[q]);
        if (q == 3) {
            if (split3) {
                append_sorted(cell_items, g->iitem_begin3, g->iitem_end3);
            } else {
                g->iitem_begin3 = g->item_begin[3];
                g->iitem_end3 = g->item_end[3];
            }
        }
    }
    if (rc == AK_OK) {
        if (AK_MALLOC(&g->items, sizeof(WorkItem) * std::max<size_t>(1, all.size())) != cudaSuccess) {
            cudaGetLastError();
            rc = fail(AK_ERR_ALLOC, "item allocation failed");
        } else if (!all.empty() &&
                   (cudaMemcpyAsync(g->items, all.data(), sizeof(WorkItem) * all.size(), cudaMemcpyHostToDevice, st) !=
                        cudaSuccess ||
                    cudaStreamSynchronize(st) != cudaSuccess)) {
            rc = fail(AK_ERR_CUDA, "item upload failed");
        }
    }
    g->nitems = (int64_t)all.size();
    if (rc == AK_OK) {
        geom_boxes(g, all, g->item_begin[3], g->item_end[3]);
        if (AK_MALLOC(&g->box_d, sizeof(int) * g->box.size()) != cudaSuccess ||
            cudaMemcpyAsync(g->box_d, g->box.data(), sizeof(int) * g->box.size(), cudaMemcpyHostToDevice, st) !=
                cudaSuccess) {
            cudaGetLastError();
            rc = fail(AK_ERR_ALLOC, "box allocation failed");
        }
    }
    if (rc == AK_OK && cached) {
        const int T = g->wf.taps;
        std::vector<int64_t> shift(P, 0);
        for (int q = 3; q >= 2 && rc == AK_OK; --q) {
            int64_t rank = 0;
            for (int w : g->windows_of_q[q]) {
                shift[w] = ((int64_t)w - rank) * N;
                const unsigned nb = (unsigned)((N + 127) / 128);
                if (q == 3)
                    k_weights<3, 12><<<nb, 128, 0, st>>>(g->pts + (int64_t)w * N, N, g->wf, g->W3 + rank * N * 3 * T,
                                                         g->CI3 + rank * N);
                else
                    k_weights<2, 12><<<nb, 128, 0, st>>>(g->pts + (int64_t)w * N, N, g->wf, g->W2 + rank * N * 2 * T,
                                                         g->CI2 + rank * N);
                if ((rc = launched()) != AK_OK) break;
                ++rank;
            }
        }
        if (rc == AK_OK) {
            if (cudaMemcpyAsync(g->wshift_d, shift.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, st) ==
                cudaSuccess) {
                g->cached = g->W3 != nullptr;
                g->cached2 = g->W2 != nullptr;
            } else {
                rc = fail(AK_ERR_CUDA, "weight table setup failed");
            }
        }
    }
    cudaStreamSynchronize(st);
    return rc;
}

static int geom_create(int32_t n, int32_t P, const int32_t* q, const int32_t* cols, const double* X, int64_t N,
                       int64_t ld, const uint8_t* masks, const int64_t* n_in, const ak_window_fn* wf,
                       const ak_tuning* tuning, void* stream, ak_geom** out);

extern "C" int ak_geom_create(int32_t n, int32_t P, const int32_t* q, const int32_t* cols, const double* X,
                              int64_t N, int64_t ld, const ak_window_fn* wf, void* stream, ak_geom** out)
{
    return geom_create(n, P, q, cols, X, N, ld, nullptr, nullptr, wf, nullptr, stream, out);
}

static int check_masks(int32_t P, int64_t N, const uint8_t* masks, const int64_t* rows_in) {
    if (!masks || !rows_in) return fail(AK_ERR_INVALID, "null argument");
    for (int w = 0; w < P; ++w)
        if (rows_in[w] < 0 || rows_in[w] > N) return fail(AK_ERR_INVALID, "bad per-window row count");
    return AK_OK;
}

extern "C" int ak_geom_create_masked(int32_t n, int32_t P, const int32_t* q, const int32_t* cols, const double* X,
                                     int64_t N, int64_t ld, const uint8_t* masks, const int64_t* rows_in,
                                     const ak_window_fn* wf, void* stream, ak_geom** out)
{
    AK_TRY(check_masks(P, N, masks, rows_in));
    return geom_create(n, P, q, cols, X, N, ld, masks, rows_in, wf, nullptr, stream, out);
}

extern "C" int ak_geom_create_ex(int32_t n, int32_t P, const int32_t* q, const int32_t* cols, const double* X,
                                 int64_t N, int64_t ld, const uint8_t* masks, const int64_t* rows_in,
                                 const ak_window_fn* wf, const ak_tuning* tuning, void* stream, ak_geom** out)
{
    if ((masks == nullptr) != (rows_in == nullptr)) return fail(AK_ERR_INVALID, "masks and rows_in go together");
    if (masks) AK_TRY(check_masks(P, N, masks, rows_in));
    if (tuning) {
        const ak_tuning& t = *tuning;
        if ((t.cell_items3 != 0 && t.cell_items3 != 1 && t.cell_items3 != 2) ||
            (t.cell_items2 != 0 && t.cell_items2 != 1 && t.cell_items2 != 8) ||
            (t.chunk3 != 0 && (t.chunk3 < 64 || t.chunk3 > 65536)) || !(t.dense_cells3 >= 0.0) ||
            !(t.dense_cells3_interp >= 0.0) || !(t.dense_cells2 >= 0.0) ||
            (t.sparse_warps != 1 && t.sparse_warps != 2) || t.tc_spread3 < 0 || t.tc_spread3 > 3)
            return fail(AK_ERR_INVALID, "bad tuning value");
    }
    return geom_create(n, P, q, cols, X, N, ld, masks, rows_in, wf, tuning, stream, out);
}

static int geom_create(int32_t n, int32_t P, const int32_t* q, const int32_t* cols, const double* X, int64_t N,
                       int64_t ld, const uint8_t* masks, const int64_t* n_in, const ak_window_fn* wf,
                       const ak_tuning* tuning, void* stream, ak_geom** out)
{
    if (!out || !q || !cols || !wf) return fail(AK_ERR_INVALID, "null argument");
    *out = nullptr;
    if (n < 2 || n > 1024) return fail(AK_ERR_INVALID, "grid size n must be in [2, 1024]");
    if (P < 1) return fail(AK_ERR_INVALID, "need at least one window");
    if (N < 0 || (N > 0 && !X)) return fail(AK_ERR_INVALID, "bad point array");
    if (N * (int64_t)P >= ((int64_t)1 << 31)) return fail(AK_ERR_INVALID, "N * P must be < 2^31");
    if (wf->taps < 4 || wf->taps > AK_MAX_TAPS || wf->taps % 2 || wf->ncoef != AK_NCOEF)
        return fail(AK_ERR_UNSUPPORTED, "window taps must be even in [4, 16] with AK_NCOEF coefficients");
    for (int w = 0; w < P; ++w) {
        if (q[w] < 1 || q[w] > 3) return fail(AK_ERR_INVALID, "window length must be 1..3");
        for (int a = 0; a < q[w]; ++a)
            if (cols[3 * w + a] < 0 || cols[3 * w + a] >= ld) return fail(AK_ERR_INVALID, "column out of range");
    }
    ak_geom* g = new ak_geom();
    g->n = n;
    g->P = P;
    g->N = N;
    g->q.assign(q, q + P);
    g->rows_in.assign(P, N);
    if (n_in) g->rows_in.assign(n_in, n_in + P);
    g->wf = *wf;
    if (tuning) g->tune = *tuning;
    else ak_tuning_default(&g->tune);
    if (wf->taps == 12) {
        bool zero = true;
        for (int k = 0; k < AK_NCOEF; ++k) zero = zero && wf->ce[0][k] == 0.0 && wf->co[0][k] == 0.0;
        g->trim3 = zero;  // taps 0 and 11 vanish: the single-cell q = 3 kernels skip them on axis 0
    }
    int rc = geom_build(g, cols, X, ld, (cudaStream_t)stream, masks, n_in);
    if (rc != AK_OK) {
        std::string keep = g_err;
        ak_geom_destroy(g);
        g_err = keep;
        return rc;
    }
    {
        char buf[256];
        const bool has3 = !g->windows_of_q[3].empty(), has2 = !g->windows_of_q[2].empty();
        snprintf(buf, sizeof buf, "q3: spread %s, interp %s, %s; q2: %s%s; taps %d%s",
                 !has3 ? "-" : (g->sedge[3] == 1 ? "cells" : "supercells 2"),
                 !has3 ? "-" : (g->sedge_i3 == 1 ? "cells" : "supercells 2"),
                 g->cached ? "weight table" : "polynomials", !has2 ? "-" : (g->sedge[2] == 1 ? "cells" : "supercells 8"),
                 has2 && g->cached2 ? " (weight table)" : "", g->wf.taps, g->tune.generic_kernels ? "; generic" : "");
        g->desc = buf;
    }
    *out = g;
    return guards_verify("ak_geom_create");
}

extern "C" const char* ak_geom_describe(const ak_geom* g) { return g ? g->desc.c_str() : ""; }

extern "C" int64_t ak_geom_num_points(const ak_geom* g) { return g ? g->N : -1; }
extern "C" int32_t ak_geom_num_windows(const ak_geom* g) { return g ? g->P : -1; }
extern "C" int64_t ak_geom_num_items(const ak_geom* g) { return g ? g->nitems : -1; }
extern "C" int64_t ak_geom_grid_elems(const ak_geom* g, int32_t w) {
    if (!g || w < 0 || w >= g->P) return -1;
    return ipow_rt(g->n, g->q[w]);
}
extern "C" int64_t ak_geom_canon_offset(const ak_geom* g, int32_t w) {
    if (!g || w < 0 || w >= g->P) return -1;
    return g->canon_off[w];
}
extern "C" int ak_geom_box(const ak_geom* g, int32_t w, int32_t* box6) {
    if (!g || !box6) return fail(AK_ERR_INVALID, "null argument");
    if (w < 0 || w >= g->P) return fail(AK_ERR_INVALID, "window out of range");
    for (int k = 0; k < 6; ++k) box6[k] = g->box[(size_t)w * 6 + k];
    return AK_OK;
}
extern "C" int64_t ak_geom_canon_total(const ak_geom* g) { return g ? g->canon_total : -1; }

// ---------------------------------------------------------------------------
// generic kernels (any taps)

namespace ak {
__global__ void k_spread_generic(const Point* __restrict__ pts, int64_t p0, int64_t np, int q,
                                 const double* __restrict__ V, Strides vs, double* __restrict__ g_w, int n,
                                 const ak_window_fn wf)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= np) return;
    const int r = blockIdx.y;
    const Point p = pts[p0 + j];
    const double v = V[(int64_t)r * vs.rs + (int64_t)p.idx * vs.is];
    double* g = g_w + (int64_t)r * (q == 3 ? (int64_t)n * n * n : (q == 2 ? (int64_t)n * n : n));
    const int T = wf.taps;
    double w[3][AK_MAX_TAPS];
    for (int a = 0; a < q; ++a)
        for (int t = 0; t < T; ++t) w[a][t] = window_weight_rt(wf, p.s[a], t);
    const int f0 = cell_axis(p.cell, 0) - (T / 2 - 1);
    const int f1 = cell_axis(p.cell, 1) - (T / 2 - 1);
    const int f2 = cell_axis(p.cell, 2) - (T / 2 - 1);
    if (q == 1) {
        for (int a = 0; a < T; ++a) red_add(g + wrap(f0 + a, n), v * w[0][a]);
    } else if (q == 2) {
        for (int a = 0; a < T; ++a) {
            const double va = v * w[0][a];
            const int64_t row = (int64_t)wrap(f0 + a, n) * n;
            for (int b = 0; b < T; ++b) red_add(g + row + wrap(f1 + b, n), va * w[1][b]);
        }
    } else {
        for (int a = 0; a < T; ++a) {
            const double va = v * w[0][a];
            const int64_t pl = (int64_t)wrap(f0 + a, n) * n;
            for (int b = 0; b < T; ++b) {
                const double vb = va * w[1][b];
                const int64_t row = (pl + wrap(f1 + b, n)) * n;
                for (int c = 0; c < T; ++c) red_add(g + row + wrap(f2 + c, n), vb * w[2][c]);
            }
        }
    }
}

__global__ void k_interp_generic(const Point* __restrict__ pts, int64_t p0, int64_t np, int q,
                                 const double* __restrict__ g_w, int n, const ak_window_fn wf,
                                 const double* __restrict__ scale, int w, double* __restrict__ out_w, Strides os,
                                 int sum_windows)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= np) return;
    const int r = blockIdx.y;
    const Point p = pts[p0 + j];
    const double* g = g_w + (int64_t)r * (q == 3 ? (int64_t)n * n * n : (q == 2 ? (int64_t)n * n : n));
    const int T = wf.taps;
    double wt[3][AK_MAX_TAPS];
    for (int a = 0; a < q; ++a)
        for (int t = 0; t < T; ++t) wt[a][t] = window_weight_rt(wf, p.s[a], t);
    const int f0 = cell_axis(p.cell, 0) - (T / 2 - 1);
    const int f1 = cell_axis(p.cell, 1) - (T / 2 - 1);
    const int f2 = cell_axis(p.cell, 2) - (T / 2 - 1);
    double acc = 0.0;
    if (q == 1) {
        for (int a = 0; a < T; ++a) acc = fma(wt[0][a], g[wrap(f0 + a, n)], acc);
    } else if (q == 2) {
        for (int a = 0; a < T; ++a) {
            const int64_t row = (int64_t)wrap(f0 + a, n) * n;
            double s = 0.0;
            for (int b = 0; b < T; ++b) s = fma(wt[1][b], g[row + wrap(f1 + b, n)], s);
            acc = fma(wt[0][a], s, acc);
        }
    } else {
        for (int a = 0; a < T; ++a) {
            const int64_t pl = (int64_t)wrap(f0 + a, n) * n;
            double sa = 0.0;
            for (int b = 0; b < T; ++b) {
                const int64_t row = (pl + wrap(f1 + b, n)) * n;
                double sb = 0.0;
                for (int c = 0; c < T; ++c) sb = fma(wt[2][c], g[row + wrap(f2 + c, n)], sb);
                sa = fma(wt[1][b], sb, sa);
            }
            acc = fma(wt[0][a], sa, acc);
        }
    }
    double* o = out_w + (int64_t)r * os.rs + (int64_t)p.idx * os.is;
    const double v = scale[w] * acc;
    if (sum_windows) red_add(o, v);
    else *o = v;
}
}  // namespace ak

// ---------------------------------------------------------------------------
// spread / interp dispatch.  Every choice is fixed at plan time (ak_geom::sedge,
// cached tables, ak_geom::tune); each launcher returns the kernel's name for the
// per-kernel timing (ak_prof_*).  Grids of every tiled launch are 1-D with the RHS
// index fastest: unit = item * R + r.

template <int Q, int T>
static const char* launch_spread_tile(const ak_geom* g, int64_t i0, int64_t ni, const double* V, Strides vs, int R,
                                      double* grids, cudaStream_t st)
{
    k_spread_tile<Q, T><<<(unsigned)(ni * R), 32, 0, st>>>(g->pts, g->items + i0, V, vs, grids, g->canon_off_d, R,
                                                           g->n, g->wf);
    return Q == 2 ? "k_spread_tile<2>" : "k_spread_tile<1>";
}

// q = 1, RHS-minor data, R >= 8: DMMA over RHS chunks (ak_q1r.cuh), RC RHS per warp
// (more than 16 RHS: chunks of 16 -- a 32-RHS chunk spills in the spread)
static int q1r_chunk(int R) { return R <= 8 ? 8 : 16; }

static const char* launch_spread1r(const ak_geom* g, int64_t i0, int64_t ni, const double* V, Strides vs, int R,
                                   double* grids, cudaStream_t st)
{
    const int rc = q1r_chunk(R);
    const dim3 grid((unsigned)(ni * AK_Q1_SPLIT_SPREAD), (unsigned)((R + rc - 1) / rc));
    if (rc == 8) k_spread1r<12, 8><<<grid, 32, 0, st>>>(g->pts, g->items + i0, V, vs, grids, g->canon_off_d, R, g->n, g->wf);
    else k_spread1r<12, 16><<<grid, 32, 0, st>>>(g->pts, g->items + i0, V, vs, grids, g->canon_off_d, R, g->n, g->wf);
    return "k_spread1r";
}

static const char* launch_interp1r(const ak_geom* g, int64_t i0, int64_t ni, const double* grids, int R,
                                   const double* scale, double* out, Strides os, int atomic_out, int64_t wstride,
                                   cudaStream_t st)
{
    const int rc = q1r_chunk(R);
    const dim3 grid((unsigned)(ni * AK_Q1_SPLIT_INTERP), (unsigned)((R + rc - 1) / rc));
    if (rc == 8)
        k_interp1r<12, 8><<<grid, 32, 0, st>>>(g->pts, g->items + i0, grids, g->canon_off_d, R, g->n, g->wf, scale,
                                               out, os, atomic_out, wstride);
    else
        k_interp1r<12, 16><<<grid, 32, 0, st>>>(g->pts, g->items + i0, grids, g->canon_off_d, R, g->n, g->wf, scale,
                                                out, os, atomic_out, wstride);
    return "k_interp1r";
}

// q = 2 single-cell items, RHS-minor data, R >= 8: 8 RHS per warp, NW warps per item
static int q2r_warps(int R) { return R <= 8 ? 1 : (R <= 16 ? 2 : 4); }

static const char* launch_spread2r(const ak_geom* g, int64_t i0, int64_t ni, const double* V, Strides vs, int R,
                                   double* grids, cudaStream_t st)
{
    const int nw = q2r_warps(R);
    const dim3 grid((unsigned)ni, (unsigned)((R + 8 * nw - 1) / (8 * nw)));
#define AK_S2R(NW) k_spread2r<AK_Q2R_SPREAD_BATCH, NW><<<grid, 32 * NW, 0, st>>>(g->CI2, g->W2, g->wshift_d, g->items + i0, V, vs, \
                                                               grids, g->canon_off_d, R, g->n)
    if (nw == 1) AK_S2R(1);
    else if (nw == 2) AK_S2R(2);
    else AK_S2R(4);
#undef AK_S2R
    return "k_spread2r";
}

static const char* launch_interp2r(const ak_geom* g, int64_t i0, int64_t ni, const double* grids, int R,
                                   const double* scale, double* out, Strides os, int atomic_out, int64_t wstride,
                                   cudaStream_t st)
{
    const int nw = q2r_warps(R);
    const dim3 grid((unsigned)ni, (unsigned)((R + 8 * nw - 1) / (8 * nw)));
#define AK_I2R(NW) k_interp2r<AK_Q2R_INTERP_BATCH, NW><<<grid, 32 * NW, 0, st>>>(g->CI2, g->W2, g->wshift_d, g->items + i0, grids, \
                                                                g->canon_off_d, R, g->n, scale, out, os, atomic_out, wstride)
    if (nw == 1) AK_I2R(1);
    else if (nw == 2) AK_I2R(2);
    else AK_I2R(4);
#undef AK_I2R
    return "k_interp2r";
}

template <int T>
static const char* launch_spread3_t(const ak_geom* g, int64_t i0, int64_t ni, const double* V, Strides vs, int R,
                                    double* grids, cudaStream_t st)
{
    const unsigned units = (unsigned)(ni * R);
    if constexpr (T == 12) {
        if (g->cached && g->sedge[3] == 1) {
            if (!g->trim3 && R % 2 == 0 && g->tune.rhs_pair_spread) {
                // pairs of RHS on the FP64 tensor cores (ak_q3r.cuh)
                k_spread3r<AK_SPREAD3R_BATCH><<<(unsigned)(ni * (R / 2)), 64, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, V,
                                                                        vs, grids, g->canon_off_d, R, g->n);
                return "k_spread3r";
            }
            if (g->trim3) {
                k_spread3c<32, 10><<<units, 32, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, V, vs, grids,
                                                         g->canon_off_d, R, g->n);
                return "k_spread3c<10>";
            }
            if (g->tune.tc_spread3 & 1) {
                k_spread3h<AK_SPREAD3H_BATCH, AK_SPREAD3H_WARPS><<<units, 32 * AK_SPREAD3H_WARPS, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, V, vs, grids,
                                                     g->canon_off_d, R, g->n);
                return "k_spread3h";
            }
            k_spread3c<32><<<units, 32, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, V, vs, grids,
                                                 g->canon_off_d, R, g->n);
            return "k_spread3c";
        }
        if (g->cached && g->sedge[3] == 2 && vs.rs == 1 && R % 8 == 0 && (g->tune.tc_spread3 & 2)) {
            // 8 RHS per CTA on the FP64 tensor cores, supercell region as the GEMM output (ak_q3b.cuh)
            static std::once_flag attr;
            std::call_once(attr, [] {
                cudaFuncSetAttribute(k_spread3b<AK_SPREAD3B_BATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)spread3b_smem<AK_SPREAD3B_BATCH>());
            });
            k_spread3b<AK_SPREAD3B_BATCH><<<(unsigned)(ni * (R / 8) * Q3B_PARTS), 32 * Q3B_WARPS, spread3b_smem<AK_SPREAD3B_BATCH>(), st>>>(
                g->CI3, g->W3, g->wshift_d, g->items + i0, V, vs, grids, g->canon_off_d, R, g->n);
            return "k_spread3b";
        }
        if (g->cached) {
            k_spread3w<12, 2, AK_SPARSE_BATCH><<<units, 32, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, V, vs, grids,
                                                        g->canon_off_d, R, g->n);
            return "k_spread3w";
        }
    }
    k_spread3<T, 2><<<units, 32, 0, st>>>(g->pts, g->items + i0, V, vs, grids, g->canon_off_d, R, g->n, g->wf);
    return "k_spread3";
}

static int spread_group(const ak_geom* g, int q, const double* V, Strides vs, int R, double* grids, cudaStream_t st) {
    const int64_t i0 = g->item_begin[q], ni = g->item_end[q] - g->item_begin[q];
    if (g->windows_of_q[q].empty() || g->N == 0) return AK_OK;
    const int T = g->wf.taps;
    const bool generic = g->tune.generic_kernels != 0;
    if (!generic && ni == 0) return AK_OK;   // only row-masked windows have no items
    if (!generic) {
        ProfScope ps(st);
        const char* name = nullptr;
        if (q == 3 && T == 12) name = launch_spread3_t<12>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 3 && T == 8) name = launch_spread3_t<8>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 3 && T == 4) name = launch_spread3_t<4>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 2 && T == 12 && g->cached2 && g->sedge[2] == 1 && vs.rs == 1 && R >= 8)
            name = launch_spread2r(g, i0, ni, V, vs, R, grids, st);
        else if (q == 2 && T == 12 && g->cached2 && g->sedge[2] == 1) {
            k_spread2c<32><<<(unsigned)(ni * R), 32, 0, st>>>(g->CI2, g->W2, g->wshift_d, g->items + i0, V, vs, grids,
                                                              g->canon_off_d, R, g->n);
            name = "k_spread2c";
        }
        else if (q == 2 && T == 12) name = launch_spread_tile<2, 12>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 2 && T == 8) name = launch_spread_tile<2, 8>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 2 && T == 16) name = launch_spread_tile<2, 16>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 2 && T == 4) name = launch_spread_tile<2, 4>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 1 && T == 12 && vs.rs == 1 && R >= 8) name = launch_spread1r(g, i0, ni, V, vs, R, grids, st);
        else if (q == 1 && T == 12) name = launch_spread_tile<1, 12>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 1 && T == 8) name = launch_spread_tile<1, 8>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 1 && T == 16) name = launch_spread_tile<1, 16>(g, i0, ni, V, vs, R, grids, st);
        else if (q == 1 && T == 4) name = launch_spread_tile<1, 4>(g, i0, ni, V, vs, R, grids, st);
        if (name) return ps.done(name);
    }
    for (int w : g->windows_of_q[q]) {
        if (g->rows_in[w] == 0) continue;
        ProfScope ps(st);
        dim3 grid((unsigned)((g->rows_in[w] + 127) / 128), (unsigned)R);
        k_spread_generic<<<grid, 128, 0, st>>>(g->pts, (int64_t)w * g->N, g->rows_in[w], q, V, vs,
                                               grids + (int64_t)R * g->canon_off[w], g->n, g->wf);
        AK_TRY(ps.done("k_spread_generic"));
    }
    return AK_OK;
}

template <int T>
static const char* launch_interp3_t(const ak_geom* g, int64_t i0, int64_t ni, const double* grids, int R,
                                    const double* scale, double* out, Strides os, int atomic_out, int64_t wstride,
                                    cudaStream_t st)
{
    const unsigned units = (unsigned)(ni * R);
    if constexpr (T == 12) {
        if (g->cached && g->sedge_i3 == 1) {
            if (g->trim3) {
                k_interp3c<32, 10><<<units, 32, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, grids,
                                                         g->canon_off_d, R, g->n, scale, out, os, atomic_out, wstride);
                return "k_interp3c<10>";
            }
            k_interp3c<AK_INTERP3C_BATCH><<<units, 32, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, grids, g->canon_off_d, R,
                                                 g->n, scale, out, os, atomic_out, wstride);
            return "k_interp3c";
        }
        if (g->cached) {
#define AK_I3M(NW) k_interp3m<2, AK_SPARSE_BATCH, NW><<<units, 32 * NW, 0, st>>>(g->CI3, g->W3, g->wshift_d, g->items + i0, grids, \
                                                                    g->canon_off_d, R, g->n, scale, out, os,          \
                                                                    atomic_out, wstride)
            if (g->tune.sparse_warps == 2) AK_I3M(2);
            else AK_I3M(1);
#undef AK_I3M
            return "k_interp3m";
        }
    }
    k_interp3<T, 2><<<units, 32, 0, st>>>(g->pts, g->items + i0, grids, g->canon_off_d, R, g->n, g->wf, scale, out, os,
                                          atomic_out, wstride);
    return "k_interp3";
}

template <int Q, int T>
static const char* launch_interp_lane(const ak_geom* g, int64_t i0, int64_t ni, const double* grids, int R,
                                      const double* scale, double* out, Strides os, int atomic_out, int64_t wstride,
                                      cudaStream_t st)
{
    k_interp_lane<Q, T><<<(unsigned)(ni * R), 32, 0, st>>>(g->pts, g->items + i0, grids, g->canon_off_d, R, g->n, g->wf,
                                                           scale, out, os, atomic_out, wstride);
    return Q == 2 ? "k_interp_lane<2>" : "k_interp_lane<1>";
}

// out(w) = out + (sum_windows ? 0 : w * wstride); atomic_out: RED instead of store
static int interp_group(const ak_geom* g, int q, const double* grids, int R, const double* scale, double* out,
                        Strides os, int sum_windows, int atomic_out, int64_t wstride, cudaStream_t st)
{
    // 3-D windows may interpolate over their own (single-cell) item list
    const int64_t i0 = q == 3 ? g->iitem_begin3 : g->item_begin[q];
    const int64_t ni = q == 3 ? g->iitem_end3 - g->iitem_begin3 : g->item_end[q] - g->item_begin[q];
    if (g->windows_of_q[q].empty() || g->N == 0) return AK_OK;
    const int T = g->wf.taps;
    const int64_t ws = sum_windows ? 0 : wstride;
    const bool generic = g->tune.generic_kernels != 0;
    if (!generic && ni == 0) return AK_OK;   // only row-masked windows have no items
    if (!generic) {
        ProfScope ps(st);
        const char* name = nullptr;
        if (q == 3 && T == 12) name = launch_interp3_t<12>(g, i0, ni, grids, R, scale, out, os, atomic_out, ws, st);
        else if (q == 3 && T == 8) name = launch_interp3_t<8>(g, i0, ni, grids, R, scale, out, os, atomic_out, ws, st);
        else if (q == 3 && T == 4) name = launch_interp3_t<4>(g, i0, ni, grids, R, scale, out, os, atomic_out, ws, st);
        else if (q == 2 && T == 12 && g->cached2 && g->sedge[2] == 1 && os.rs == 1 && R >= 8)
            name = launch_interp2r(g, i0, ni, grids, R, scale, out, os, atomic_out, ws, st);
        else if (q == 2 && T == 12 && g->cached2 && g->sedge[2] == 1) {
            k_interp2c<32><<<(unsigned)(ni * R), 32, 0, st>>>(g->CI2, g->W2, g->wshift_d, g->items + i0, grids,
                                                              g->canon_off_d, R, g->n, scale, out, os, atomic_out, ws);
            name = "k_interp2c";
        }
        else if (q == 1 && T == 12 && os.rs == 1 && R >= 8)
            name = launch_interp1r(g, i0, ni, grids, R, scale, out, os, atomic_out, ws, st);
#define AK_LANE(QQ, TT) \
        else if (q == QQ && T == TT) name = launch_interp_lane<QQ, TT>(g, i0, ni, grids, R, scale, out, os, atomic_out, ws, st);
        AK_LANE(2, 4) AK_LANE(2, 6) AK_LANE(2, 8) AK_LANE(2, 10) AK_LANE(2, 12) AK_LANE(2, 14) AK_LANE(2, 16)
        AK_LANE(1, 4) AK_LANE(1, 6) AK_LANE(1, 8) AK_LANE(1, 10) AK_LANE(1, 12) AK_LANE(1, 14) AK_LANE(1, 16)
#undef AK_LANE
        if (name) return ps.done(name);
    }
    for (int w : g->windows_of_q[q]) {
        if (g->rows_in[w] == 0) continue;
        ProfScope ps(st);
        dim3 grid((unsigned)((g->rows_in[w] + 127) / 128), (unsigned)R);
        k_interp_generic<<<grid, 128, 0, st>>>(g->pts, (int64_t)w * g->N, g->rows_in[w], q,
                                               grids + (int64_t)R * g->canon_off[w],
                                               g->n, g->wf, scale, w, out + (int64_t)w * ws, os, atomic_out);
        AK_TRY(ps.done("k_interp_generic"));
    }
    return AK_OK;
}

// Launch-shape limits: RHS on grid.y (<= 65535) or folded into grid.x with the items.
static int check_rhs(const ak_geom* g, int R) {
    if (R > 65535 || g->nitems * (int64_t)R >= ((int64_t)1 << 31))
        return fail(AK_ERR_UNSUPPORTED, "too many right-hand sides for one call (R <= 65535, items x R < 2^31)");
    return AK_OK;
}

extern "C" int ak_spread(const ak_geom* g, const double* V, int32_t R, int64_t ldv, double* grids, void* stream) {
    if (!g || R < 1 || (g->N > 0 && (!V || !grids)) || ldv < g->N) return fail(AK_ERR_INVALID, "bad spread arguments");
    AK_TRY(check_rhs(g, R));
    cudaStream_t st = (cudaStream_t)stream;
    for (int q = 3; q >= 1; --q) AK_TRY(spread_group(g, q, V, Strides{ldv, 1}, R, grids, st));
    return guards_verify("ak_spread");
}

extern "C" int ak_interp(const ak_geom* g, const double* grids, int32_t R, const double* scale, double* out,
                         int64_t ldo, int32_t sum_windows, int64_t wstride, void* stream)
{
    if (!g || R < 1 || !scale || (g->N > 0 && (!grids || !out)) || ldo < g->N)
        return fail(AK_ERR_INVALID, "bad interp arguments");
    AK_TRY(check_rhs(g, R));
    cudaStream_t st = (cudaStream_t)stream;
    for (int q = 3; q >= 1; --q)
        AK_TRY(interp_group(g, q, grids, R, scale, out, Strides{ldo, 1}, sum_windows, sum_windows ? 1 : 0, wstride,
                            st));
    return guards_verify("ak_interp");
}

// ---------------------------------------------------------------------------
// FFT stage

// Y2 = H (compact band multiplier of the window) * Y on the band, 0 elsewhere.
__global__ void k_band_multiply(const double2* __restrict__ Y, double2* __restrict__ Y2, int q, int n, int m,
                                int R, int64_t hs, int64_t total, const int* __restrict__ gwin,
                                const double* const* __restrict__ H, int hbase, int P, int per_rhs)
{
    const int nh = n / 2 + 1, mh = m / 2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / hs;
        const int64_t k = e - b * hs;
        const int k2 = (int)(k % nh);
        const int64_t rest = k / nh;
        int k0 = 0, k1 = 0;
        if (q == 3) {
            k1 = (int)(rest % n);
            k0 = (int)(rest / n);
        } else if (q == 2) {
            k1 = (int)rest;
        }
        bool in = k2 < mh;
        int b0 = 0, b1 = 0;
        if (q >= 2) {
            in = in && (k1 < mh || k1 >= n - mh);
            b1 = k1 < mh ? k1 : k1 - (n - m);
        }
        if (q == 3) {
            in = in && (k0 < mh || k0 >= n - mh);
            b0 = k0 < mh ? k0 : k0 - (n - m);
        }
        double2 out = make_double2(0.0, 0.0);
        if (in) {
            const int w = gwin[b / R];
            const int hsel = per_rhs ? (int)(b % R) * P + w : hbase + w;
            int64_t ci;
            if (q == 3) ci = ((int64_t)b0 * m + b1) * mh + k2;
            else if (q == 2) ci = (int64_t)b1 * mh + k2;
            else ci = k2;
            const double h = H[hsel][ci];
            const double2 y = Y[e];
            out = make_double2(h * y.x, h * y.y);
        }
        Y2[e] = out;
    }
}

// Band of the half spectra <-> compact exchange buffer (same compact indexing as H):
// dir = 0 packs spec -> band, dir = 1 unpacks band -> spec (band entries only).
__global__ void k_band_pack(double2* __restrict__ spec, double2* __restrict__ band, int q, int n, int m, int64_t hs,
                            int64_t bs, int64_t total, int dir)
{
    const int nh = n / 2 + 1, mh = m / 2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / bs;
        const int64_t k = e - b * bs;
        const int k2 = (int)(k % mh);
        const int64_t rest = k / mh;
        int64_t lin;
        if (q == 3) {
            const int b1 = (int)(rest % m), b0 = (int)(rest / m);
            const int k0 = b0 < mh ? b0 : b0 + (n - m), k1 = b1 < mh ? b1 : b1 + (n - m);
            lin = ((int64_t)k0 * n + k1) * nh + k2;
        } else if (q == 2) {
            const int b1 = (int)rest;
            const int k1 = b1 < mh ? b1 : b1 + (n - m);
            lin = (int64_t)k1 * nh + k2;
        } else {
            lin = k2;
        }
        if (dir == 0) band[e] = spec[b * hs + lin];
        else spec[b * hs + lin] = band[e];
    }
}

// The fused 3-D transform stage is compiled for the default and rough presets at the
// default oversampling (n, m) = (64, 32), (32, 16); other shapes (and a geometry with
// ak_tuning::fused_fft3 = 0) use the full cuFFT transforms.
template <int n, int m>
static void fft3_attrs() {
    cudaFuncSetAttribute(ak::k_fft3_fwd12<n, m>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ak::fft3_smem_fwd12(n, m));
    cudaFuncSetAttribute(ak::k_fft3_fwd0<n, m>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ak::fft3_smem_fwd0(n, m));
    cudaFuncSetAttribute(ak::k_fft3_inv0<n, m>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ak::fft3_smem_inv0(n, m));
    cudaFuncSetAttribute(ak::k_fft3_inv12<n, m>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ak::fft3_smem_inv12(n, m));
}

static bool fft3_fused_ok(const ak_geom* g, int n, int m) {
    if (!g->tune.fused_fft3) return false;
    if (n == 64 && m == 32) fft3_attrs<64, 32>();
    else if (n == 32 && m == 16) fft3_attrs<32, 16>();
    else return false;
    return true;
}

struct ak_op;
static int fft3_forward(ak_op* op, bool full_box, cudaStream_t st);
static int fft3_inverse(ak_op* op, const double* const* H, int hbase, int per_rhs, cudaStream_t st);

struct ak_op {
    const ak_geom* gs = nullptr;
    const ak_geom* gi = nullptr;
    int m = 0, R = 0, C = 0;
    double* grids = nullptr;      // canonical, R rhs
    double* gbuf = nullptr;       // canonical, R rhs
    double2* spec = nullptr;
    double2* spec2 = nullptr;
    int64_t spec_off[4] = {0, 0, 0, 0};   // complex elements, per q group
    double2* band = nullptr;              // compact band spectra (multi-GPU exchange buffer)
    int64_t band_off[4] = {0, 0, 0, 0};
    int64_t bs[4] = {0, 0, 0, 0};         // band elements per grid
    int64_t band_total = 0;
    int64_t hs[4] = {0, 0, 0, 0};         // half-spectrum elements per grid
    int64_t grid_off[4] = {0, 0, 0, 0};   // doubles, per q group (R units applied)
    int nwin[4] = {0, 0, 0, 0};
    cufftHandle fwd[4] = {0, 0, 0, 0}, inv[4] = {0, 0, 0, 0};
    bool has[4] = {false, false, false, false};
    bool planned[4] = {false, false, false, false};   // cuFFT plans made for this q
    bool fused3 = false;          // q = 3: band-pruned fused transforms (ak_fft3.cuh) instead of cuFFT
    double* fbuf = nullptr;       // fused3: per-plane partial transforms [R nwin3][n][2][m][m/2]
    double* ftab = nullptr;       // fused3: twiddle tables (ak::Fft3Tables)
    int* gwin_d[4] = {nullptr, nullptr, nullptr, nullptr};
};

static ak::Fft3Tables fft3_tables(const ak_op* op) {
    const size_t nm = (size_t)op->gs->n * op->m;
    const double* t = op->ftab;
    return ak::Fft3Tables{t, t + nm, t + 2 * nm, t + 6 * nm};
}

// largest box extent along axis 0 over the 3-D windows (the launches' plane count)
static int box_planes(const ak_geom* g) {
    int L0 = 0;
    for (int w : g->windows_of_q[3]) L0 = std::max(L0, g->box[(size_t)w * 6 + 1]);
    return std::max(L0, 1);
}

// fused q = 3 transforms: grids -> compact band spectra (op->band, q = 3 section).
// full_box: the grids hold more than this op's spread (AK_APPLY_FROM_GRIDS after a
// grid all-reduce): transform whole grids instead of the spread geometry's boxes.
template <int n, int m>
static int fft3_forward_t(ak_op* op, bool full_box, cudaStream_t st) {
    const unsigned nb = (unsigned)(op->R * op->nwin[3]);
    const ak::Fft3Tables tb = fft3_tables(op);
    const int* box = full_box ? nullptr : op->gs->box_d;
    const unsigned planes = full_box ? (unsigned)n : (unsigned)box_planes(op->gs);
    {
        ProfScope ps(st);
        ak::k_fft3_fwd12<n, m><<<dim3(planes, nb), ak::FFT3_THREADS, ak::fft3_smem_fwd12(n, m), st>>>(
            op->grids + op->grid_off[3], op->fbuf, tb, box, op->gwin_d[3], op->R);
        AK_TRY(ps.done("k_fft3_fwd12"));
    }
    ProfScope ps(st);
    ak::k_fft3_fwd0<n, m><<<dim3(m, nb), ak::FFT3_THREADS, ak::fft3_smem_fwd0(n, m), st>>>(
        op->fbuf, reinterpret_cast<double*>(op->band + op->band_off[3]), tb, box, op->gwin_d[3], op->R);
    return ps.done("k_fft3_fwd0");
}

// fused q = 3: H (set hbase / per RHS) x band spectra -> the interpolation geometry's
// boxes of the op->gbuf grids
template <int n, int m>
static int fft3_inverse_t(ak_op* op, const double* const* H, int hbase, int per_rhs, cudaStream_t st) {
    const unsigned nb = (unsigned)(op->R * op->nwin[3]);
    const ak::Fft3Tables tb = fft3_tables(op);
    const int* box = op->gi->box_d;
    {
        ProfScope ps(st);
        ak::k_fft3_inv0<n, m><<<dim3(m, nb), ak::FFT3_THREADS, ak::fft3_smem_inv0(n, m), st>>>(
            reinterpret_cast<const double*>(op->band + op->band_off[3]), op->fbuf, tb, op->R, op->gwin_d[3], H, hbase,
            op->gs->P, per_rhs, box);
        AK_TRY(ps.done("k_fft3_inv0"));
    }
    ProfScope ps(st);
    ak::k_fft3_inv12<n, m><<<dim3((unsigned)box_planes(op->gi), nb), ak::FFT3_THREADS, ak::fft3_smem_inv12(n, m), st>>>(
        op->fbuf, op->gbuf + op->grid_off[3], tb, box, op->gwin_d[3], op->R);
    return ps.done("k_fft3_inv12");
}

static int fft3_forward(ak_op* op, bool full_box, cudaStream_t st) {
    return op->gs->n == 64 ? fft3_forward_t<64, 32>(op, full_box, st) : fft3_forward_t<32, 16>(op, full_box, st);
}

static int fft3_inverse(ak_op* op, const double* const* H, int hbase, int per_rhs, cudaStream_t st) {
    return op->gs->n == 64 ? fft3_inverse_t<64, 32>(op, H, hbase, per_rhs, st)
                           : fft3_inverse_t<32, 16>(op, H, hbase, per_rhs, st);
}

extern "C" int ak_op_destroy(ak_op* op) {
    if (!op) return AK_OK;
    for (int q = 1; q <= 3; ++q) {
        if (op->planned[q]) {
            cufftDestroy(op->fwd[q]);
            cufftDestroy(op->inv[q]);
        }
        ak_free(op->gwin_d[q]);
    }
    ak_free(op->fbuf);
    ak_free(op->ftab);
    ak_free(op->grids);
    ak_free(op->gbuf);
    ak_free(op->spec);
    ak_free(op->spec2);
    ak_free(op->band);
    delete op;
    return AK_OK;
}

static int op_build(ak_op* op, cudaStream_t st) {
    const ak_geom* g = op->gs;
    const int n = g->n;
    const int64_t total = g->canon_total * op->R;
    AK_CUDA(AK_MALLOC(&op->grids, sizeof(double) * total));
    AK_CUDA(AK_MALLOC(&op->gbuf, sizeof(double) * total));
    int64_t soff = 0;
    for (int q = 3; q >= 1; --q) {
        const auto& ws = g->windows_of_q[q];
        op->nwin[q] = (int)ws.size();
        op->hs[q] = ipow_rt(n, q - 1) * (n / 2 + 1);
        op->spec_off[q] = soff;
        if (ws.empty()) continue;
        op->grid_off[q] = (int64_t)op->R * g->canon_off[ws[0]];
        AK_CUDA(AK_MALLOC(&op->gwin_d[q], sizeof(int) * ws.size()));
        AK_CUDA(cudaMemcpyAsync(op->gwin_d[q], ws.data(), sizeof(int) * ws.size(), cudaMemcpyHostToDevice, st));
        op->has[q] = true;
        const int batch = op->R * (int)ws.size();
        if (q == 3 && batch <= 65535 && fft3_fused_ok(g, n, op->m)) {   // grids on gridDim.y
            op->fused3 = true;
            AK_CUDA(AK_MALLOC(&op->fbuf, sizeof(double) * (size_t)batch * n * op->m * op->m));
            const std::vector<double> tabs = ak::fft3_host_tables(n, op->m);
            AK_CUDA(AK_MALLOC(&op->ftab, sizeof(double) * tabs.size()));
            AK_CUDA(cudaMemcpyAsync(op->ftab, tabs.data(), sizeof(double) * tabs.size(), cudaMemcpyHostToDevice, st));
            AK_CUDA(cudaStreamSynchronize(st));
            continue;
        }
        soff += op->hs[q] * batch;
        int dims[3] = {n, n, n};
        AK_CUFFT(cufftPlanMany(&op->fwd[q], q, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, batch));
        if (cufftPlanMany(&op->inv[q], q, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, batch) != CUFFT_SUCCESS) {
            cufftDestroy(op->fwd[q]);
            return fail(AK_ERR_CUFFT, "cufftPlanMany Z2D failed");
        }
        op->planned[q] = true;
    }
    int64_t boff = 0;
    for (int q = 3; q >= 1; --q) {
        op->bs[q] = ipow_rt(op->m, q - 1) * (op->m / 2);
        op->band_off[q] = boff;
        boff += op->bs[q] * op->R * op->nwin[q];
    }
    op->band_total = boff;
    AK_CUDA(AK_MALLOC(&op->band, sizeof(double2) * std::max<int64_t>(boff, 1)));
    AK_CUDA(AK_MALLOC(&op->spec, sizeof(double2) * std::max<int64_t>(soff, 1)));
    AK_CUDA(AK_MALLOC(&op->spec2, sizeof(double2) * std::max<int64_t>(soff, 1)));
    AK_CUDA(cudaStreamSynchronize(st));
    return AK_OK;
}

extern "C" int ak_op_create(const ak_geom* spread_geom, const ak_geom* interp_geom, int32_t m, int32_t R, int32_t C,
                            void* stream, ak_op** out)
{
    if (!out || !spread_geom) return fail(AK_ERR_INVALID, "null argument");
    *out = nullptr;
    if (!interp_geom) interp_geom = spread_geom;
    if (R < 1 || C < 1) return fail(AK_ERR_INVALID, "R and C must be >= 1");
    if (m < 2 || m % 2 || m > spread_geom->n) return fail(AK_ERR_INVALID, "m must be even, 2 <= m <= n");
    if (interp_geom->n != spread_geom->n || interp_geom->q != spread_geom->q)
        return fail(AK_ERR_INVALID, "spread and interp geometries must share windows and n");
    AK_TRY(check_rhs(spread_geom, R));
    AK_TRY(check_rhs(interp_geom, R));
    ak_op* op = new ak_op();
    op->gs = spread_geom;
    op->gi = interp_geom;
    op->m = m;
    op->R = R;
    op->C = C;
    int rc = op_build(op, (cudaStream_t)stream);
    if (rc != AK_OK) {
        std::string keep = g_err;
        ak_op_destroy(op);
        g_err = keep;
        return rc;
    }
    *out = op;
    return AK_OK;
}

extern "C" int ak_op_grids(ak_op* op, double** grids, int64_t* count) {
    if (!op || !grids || !count) return fail(AK_ERR_INVALID, "null argument");
    *grids = op->grids;
    *count = op->gs->canon_total * op->R;
    return AK_OK;
}

extern "C" int ak_op_band(ak_op* op, double** band, int64_t* count) {
    if (!op || !band || !count) return fail(AK_ERR_INVALID, "null argument");
    *band = reinterpret_cast<double*>(op->band);
    *count = 2 * op->band_total;
    return AK_OK;
}

// cuFFT transform of one window-length group, timed as one "kernel" when profiling
static int cufft_d2z(ak_op* op, int q, cudaStream_t st) {
    ProfScope ps(st);
    AK_CUFFT(cufftSetStream(op->fwd[q], st));
    AK_CUFFT(cufftExecD2Z(op->fwd[q], op->grids + op->grid_off[q], (cufftDoubleComplex*)(op->spec + op->spec_off[q])));
    g_launches.fetch_add(1);
    ps.close(q == 3 ? "cufft_d2z<3>" : (q == 2 ? "cufft_d2z<2>" : "cufft_d2z<1>"));
    return AK_OK;
}

static int band_pack(ak_op* op, int q, int dir, cudaStream_t st) {
    ProfScope ps(st);
    const int64_t total = op->bs[q] * op->R * op->nwin[q];
    k_band_pack<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
        op->spec + op->spec_off[q], op->band + op->band_off[q], q, op->gs->n, op->m, op->hs[q], op->bs[q], total, dir);
    return ps.done("k_band_pack");
}

static int op_apply(ak_op* op, const double* V, int64_t ldv, const double* const* H, const double* scale,
                    double* const* outs, int64_t ldo, const int32_t* sum_windows, int32_t flags, void* stream);

extern "C" int ak_op_apply(ak_op* op, const double* V, int64_t ldv, const double* const* H, const double* scale,
                           double* const* outs, int64_t ldo, const int32_t* sum_windows, int32_t flags,
                           void* stream)
{
    const int rc = op_apply(op, V, ldv, H, scale, outs, ldo, sum_windows, flags, stream);
#ifdef AK_CHECKED
    // (no device synchronisation while the caller captures a CUDA graph: the guard
    // bands are verified at the next uncaptured entry point)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing((cudaStream_t)stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return rc;
#endif
    return rc == AK_OK ? guards_verify("ak_op_apply") : rc;
}

static int op_apply(ak_op* op, const double* V, int64_t ldv, const double* const* H, const double* scale,
                    double* const* outs, int64_t ldo, const int32_t* sum_windows, int32_t flags, void* stream)
{
    if (!op) return fail(AK_ERR_INVALID, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const ak_geom* gs = op->gs;
    const ak_geom* gi = op->gi;
    const int R = op->R, P = gs->P;
    const int accumulate = flags & AK_APPLY_ACCUMULATE;
    const bool minor = (flags & AK_APPLY_RHS_MINOR) != 0;
    if (!(flags & (AK_APPLY_FROM_GRIDS | AK_APPLY_FROM_SPECTRUM))) {
        if ((minor ? ldv < R : ldv < gs->N) || (gs->N > 0 && !V)) return fail(AK_ERR_INVALID, "bad right-hand sides");
        const Strides vs = minor ? Strides{1, ldv} : Strides{ldv, 1};
        AK_CUDA(cudaMemsetAsync(op->grids, 0, sizeof(double) * gs->canon_total * R, st));
        if (gs->N > 0)
            for (int q = 3; q >= 1; --q) AK_TRY(spread_group(gs, q, V, vs, R, op->grids, st));
    }
    if (flags & AK_APPLY_SPREAD_ONLY) return AK_OK;
    if (flags & AK_APPLY_SPECTRUM_ONLY) {
        for (int q = 3; q >= 1; --q)
            if (q == 3 && op->fused3) {
                AK_TRY(fft3_forward(op, false, st));
            } else if (op->has[q]) {
                AK_TRY(cufft_d2z(op, q, st));
                AK_TRY(band_pack(op, q, 0, st));
            }
        return AK_OK;
    }
    if (!H || !scale || !outs || !sum_windows) return fail(AK_ERR_INVALID, "null argument");
    if (minor ? ldo < R : ldo < gi->N) return fail(AK_ERR_INVALID, "leading dimension too small");
    if ((flags & AK_APPLY_H_PER_RHS) && op->C != 1) return fail(AK_ERR_INVALID, "per-RHS multipliers need C == 1");
    // RHS-major: summed out[r*ldo + i], per window out[(w*R + r)*ldo + i];
    // RHS-minor: summed out[i*ldo + r], per window out[(w*N + i)*ldo + r]
    const Strides os = minor ? Strides{1, ldo} : Strides{ldo, 1};
    const int64_t wstride = minor ? gi->N * ldo : (int64_t)R * ldo;
    for (int c = 0; c < op->C; ++c) {
        if (!outs[c]) return fail(AK_ERR_INVALID, "null output");
        if (!accumulate) {
            const int64_t one = minor ? gi->N * ldo : (int64_t)R * ldo;
            AK_CUDA(cudaMemsetAsync(outs[c], 0, sizeof(double) * one * (sum_windows[c] ? 1 : P), st));
        }
    }
    if (gi->N == 0) return AK_OK;
    for (int q = 3; q >= 1; --q)
        if (q == 3 && op->fused3) {
            // the band spectrum is the fused stage's intermediate: from-spectrum starts at the inverse
            if (!(flags & AK_APPLY_FROM_SPECTRUM)) AK_TRY(fft3_forward(op, (flags & AK_APPLY_FROM_GRIDS) != 0, st));
        } else if (op->has[q]) {
            if (flags & AK_APPLY_FROM_SPECTRUM) AK_TRY(band_pack(op, q, 1, st));
            else AK_TRY(cufft_d2z(op, q, st));
        }
    for (int c = 0; c < op->C; ++c) {
        for (int q = 3; q >= 1; --q) {
            if (!op->has[q]) continue;
            if (q == 3 && op->fused3) {
                AK_TRY(fft3_inverse(op, H, c * P, (flags & AK_APPLY_H_PER_RHS) ? 1 : 0, st));
                continue;
            }
            const int64_t total = op->hs[q] * R * op->nwin[q];
            const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
            {
                ProfScope ps(st);
                k_band_multiply<<<blocks, 256, 0, st>>>(op->spec + op->spec_off[q], op->spec2 + op->spec_off[q], q,
                                                        gs->n, op->m, R, op->hs[q], total, op->gwin_d[q], H, c * P, P,
                                                        (flags & AK_APPLY_H_PER_RHS) ? 1 : 0);
                AK_TRY(ps.done("k_band_multiply"));
            }
            ProfScope ps(st);
            AK_CUFFT(cufftSetStream(op->inv[q], st));
            AK_CUFFT(cufftExecZ2D(op->inv[q], (cufftDoubleComplex*)(op->spec2 + op->spec_off[q]),
                                  op->gbuf + op->grid_off[q]));
            g_launches.fetch_add(1);
            ps.close(q == 3 ? "cufft_z2d<3>" : (q == 2 ? "cufft_z2d<2>" : "cufft_z2d<1>"));
        }
        const int atomic_out = (sum_windows[c] || accumulate) ? 1 : 0;
        for (int q = 3; q >= 1; --q)
            AK_TRY(interp_group(gi, q, op->gbuf, R, scale + (int64_t)c * P, outs[c], os, sum_windows[c], atomic_out,
                                wstride, st));
    }
    return AK_OK;
}

// ---------------------------------------------------------------------------
// complex NUFFT building blocks

// Plans are cached per (shape, type, stream): a cuFFT plan owns one work area, so
// one plan must not execute on two streams at once.
struct PlanKey {
    int q, n, type;
    cudaStream_t stream;
    bool operator<(const PlanKey& o) const {
        return std::tie(q, n, type, stream) < std::tie(o.q, o.n, o.type, o.stream);
    }
};
static std::mutex g_plan_mu;
static std::map<PlanKey, cufftHandle> g_plans;

// At most kMaxCachedPlans (shape, type, stream) plans are kept; beyond that (a process
// cycling through many streams) a call gets a temporary plan that the caller destroys
// after synchronising its stream.
static constexpr size_t kMaxCachedPlans = 64;

static int cached_plan(int q, int n, cufftType type, cudaStream_t st, cufftHandle* out, bool* temporary) {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    PlanKey k{q, n, (int)type, st};
    *temporary = false;
    auto it = g_plans.find(k);
    if (it != g_plans.end()) {
        *out = it->second;
        return AK_OK;
    }
    int dims[3] = {n, n, n};
    cufftHandle h;
    AK_CUFFT(cufftPlanMany(&h, q, dims, nullptr, 1, 0, nullptr, 1, 0, type, 1));
    if (cufftSetStream(h, st) != CUFFT_SUCCESS) {
        cufftDestroy(h);
        return fail(AK_ERR_CUFFT, "cufftSetStream failed");
    }
    if (g_plans.size() < kMaxCachedPlans) g_plans[k] = h;
    else *temporary = true;
    *out = h;
    return AK_OK;
}

// Release a plan obtained with *temporary set, once the work queued on `st` is done.
static void release_plan(cufftHandle h, bool temporary, cudaStream_t st) {
    if (!temporary) return;
    cudaStreamSynchronize(st);
    cufftDestroy(h);
}

__global__ void k_type1_extract(const double2* __restrict__ Yr, const double2* __restrict__ Yi, int q, int n, int m,
                                const double* __restrict__ deconv, double2* __restrict__ S)
{
    const int64_t tot = q == 3 ? (int64_t)m * m * m : (q == 2 ? (int64_t)m * m : m);
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= tot) return;
    int ja[3] = {0, 0, 0};
    int64_t rest = j;
    for (int a = q - 1; a >= 0; --a) {
        ja[a] = (int)(rest % m);
        rest /= m;
    }
    int kn[3];
    double dc = 1.0;
    for (int a = 0; a < q; ++a) {
        const int k = ja[a] < m / 2 ? ja[a] : ja[a] - m;
        kn[a] = k >= 0 ? k : k + n;
        dc *= deconv[a * m + ja[a]];
    }
    const int nh = n / 2 + 1;
    bool conj = kn[q - 1] > n / 2;
    int idx[3];
    for (int a = 0; a < q; ++a) idx[a] = conj ? (n - kn[a]) % n : kn[a];
    int64_t lin = 0;
    for (int a = 0; a < q; ++a) lin = lin * (a == q - 1 ? nh : n) + idx[a];
    double2 yr = Yr[lin], yi = Yi[lin];
    if (conj) {
        yr.y = -yr.y;
        yi.y = -yi.y;
    }
    S[j] = make_double2(dc * (yr.x - yi.y), dc * (yr.y + yi.x));
}

extern "C" int ak_type1_band(int32_t q, int32_t n, int32_t m, const double* gre, const double* gim,
                             const double* deconv, double* S, void* stream)
{
    if (q < 1 || q > 3 || m < 2 || m > n || !gre || !gim || !deconv || !S) return fail(AK_ERR_INVALID, "bad type1 args");
    cudaStream_t st = (cudaStream_t)stream;
    cufftHandle h;
    bool tmp_plan = false;
    AK_TRY(cached_plan(q, n, CUFFT_D2Z, st, &h, &tmp_plan));
    const int64_t hs = ipow_rt(n, q - 1) * (n / 2 + 1);
    double2* Y = nullptr;
    if (cudaMallocAsync(&Y, sizeof(double2) * hs * 2, st) != cudaSuccess) {
        cudaGetLastError();
        release_plan(h, tmp_plan, st);
        return fail(AK_ERR_ALLOC, "type-1 workspace allocation failed");
    }
    int rc = AK_OK;
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        if (cufftExecD2Z(h, const_cast<double*>(gre), (cufftDoubleComplex*)Y) != CUFFT_SUCCESS ||
            cufftExecD2Z(h, const_cast<double*>(gim), (cufftDoubleComplex*)(Y + hs)) != CUFFT_SUCCESS)
            rc = fail(AK_ERR_CUFFT, "cufftExecD2Z failed");
    }
    if (rc == AK_OK) {
        g_launches.fetch_add(2);
        const int64_t tot = ipow_rt(m, q);
        k_type1_extract<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Y, Y + hs, q, n, m, deconv, (double2*)S);
        rc = launched();
    }
    cudaFreeAsync(Y, st);
    release_plan(h, tmp_plan, st);
    return rc == AK_OK ? guards_verify("ak_type1_band") : rc;
}

__global__ void k_type2_pad(const double2* __restrict__ c, int q, int n, int m, const double* __restrict__ deconv,
                            double2* __restrict__ G)
{
    const int64_t tot = q == 3 ? (int64_t)m * m * m : (q == 2 ? (int64_t)m * m : m);
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= tot) return;
    int ja[3] = {0, 0, 0};
    int64_t rest = j;
    for (int a = q - 1; a >= 0; --a) {
        ja[a] = (int)(rest % m);
        rest /= m;
    }
    double dc = 1.0;
    int64_t lin = 0;
    for (int a = 0; a < q; ++a) {
        const int k = ja[a] < m / 2 ? ja[a] : ja[a] - m;
        lin = lin * n + (k >= 0 ? k : k + n);
        dc *= deconv[a * m + ja[a]];
    }
    const double2 v = c[j];
    G[lin] = make_double2(dc * v.x, dc * v.y);
}

__global__ void k_split(const double2* __restrict__ G, int64_t tot, double* __restrict__ re, double* __restrict__ im) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= tot) return;
    const double2 v = G[i];
    re[i] = v.x;
    im[i] = v.y;
}

extern "C" int ak_type2_grid(int32_t q, int32_t n, int32_t m, const double* c, const double* deconv, double* gre,
                             double* gim, void* stream)
{
    if (q < 1 || q > 3 || m < 2 || m > n || !c || !deconv || !gre || !gim) return fail(AK_ERR_INVALID, "bad type2 args");
    cudaStream_t st = (cudaStream_t)stream;
    cufftHandle h;
    bool tmp_plan = false;
    AK_TRY(cached_plan(q, n, CUFFT_Z2Z, st, &h, &tmp_plan));
    const int64_t tot = ipow_rt(n, q);
    double2* G = nullptr;
    if (cudaMallocAsync(&G, sizeof(double2) * tot, st) != cudaSuccess) {
        cudaGetLastError();
        release_plan(h, tmp_plan, st);
        return fail(AK_ERR_ALLOC, "type-2 workspace allocation failed");
    }
    int rc = cudaMemsetAsync(G, 0, sizeof(double2) * tot, st) == cudaSuccess ? AK_OK
                                                                               : fail(AK_ERR_CUDA, "memset failed");
    if (rc == AK_OK) {
        const int64_t tm = ipow_rt(m, q);
        k_type2_pad<<<(unsigned)((tm + 255) / 256), 256, 0, st>>>((const double2*)c, q, n, m, deconv, G);
        rc = launched();
    }
    if (rc == AK_OK) {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        if (cufftExecZ2Z(h, (cufftDoubleComplex*)G, (cufftDoubleComplex*)G, CUFFT_INVERSE) != CUFFT_SUCCESS)
            rc = fail(AK_ERR_CUFFT, "cufftExecZ2Z failed");
        else
            g_launches.fetch_add(1);
    }
    if (rc == AK_OK) {
        k_split<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(G, tot, gre, gim);
        rc = launched();
    }
    cudaFreeAsync(G, st);
    release_plan(h, tmp_plan, st);
    return rc == AK_OK ? guards_verify("ak_type2_grid") : rc;
}
