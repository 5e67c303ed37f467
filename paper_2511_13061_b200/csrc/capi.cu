// capi.cu — host runtime and the extern "C" boundary of libmacko_cuda.so (include/macko_cuda.h).
//
// Owns device matrices (values / packed deltas / row pointers in the reference byte layout,
// matrix.hpp:57-81), builds the static SpMV work plan once per matrix, drives the compressor
// and maps every failure onto a status code + thread-local message (no exception crosses the
// C boundary; the C++ wrapper include/macko/macko_cuda.hpp rethrows the reference types).
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <new>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/macko_cuda.h"
#include "common.cuh"
#include "compress.cuh"
#include "plan.cuh"
#include "spmv.cuh"

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<uint32_t> g_trace_slot{0};  // trace builds: round-robin slot of each SpMV launch

struct Failure {
    macko_status code;
    std::string msg;
};

[[noreturn]] void fail(macko_status code, const std::string& msg) { throw Failure{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    cudaGetLastError();  // clear sticky-less errors
    fail(e == cudaErrorMemoryAllocation ? MACKO_ENOMEM : MACKO_ECUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
macko_status guarded(F&& f) {
    try {
        f();
        return MACKO_OK;
    } catch (const Failure& x) {
        g_err = x.msg;
        return x.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return MACKO_ENOMEM;
    } catch (...) {
        g_err = "unknown failure";
        return MACKO_ECUDA;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        ck(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// Device block cache behind DevBuf.  cudaMalloc / cudaFree of the compressor's buffers (566 MB of
// values + codewords at 36864x12288, plus scratch) cost milliseconds per build; released blocks of
// >= 1 MiB are kept per device (up to kCacheBytes) and reused for a request of 50-100 % of their
// size.  A release still synchronises the device first, exactly as cudaFree does, so a block is
// never handed out while an earlier kernel may use it.  macko_release_cached_memory() frees them.
class BlockCache {
  public:
    static constexpr size_t kMinBytes = 1u << 20, kCacheBytes = size_t(4) << 30;
    const bool off = std::getenv("MACKO_NO_BLOCK_CACHE") != nullptr;  // A/B switch
    void* get(int dev, size_t bytes) {
        if (bytes >= kMinBytes && !off) {
            std::lock_guard<std::mutex> lk(mu_);
            auto best = blocks_.end();
            for (auto it = blocks_.begin(); it != blocks_.end(); ++it)
                if (it->dev == dev && it->bytes >= bytes && it->bytes <= 2 * bytes &&
                    (best == blocks_.end() || it->bytes < best->bytes))
                    best = it;
            if (best != blocks_.end()) {
                void* p = best->p;
                held_ -= best->bytes;
                live_[p] = best->bytes;
                blocks_.erase(best);
                return p;
            }
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {  // out of memory: drop the cache and retry once
            cudaGetLastError();
            trim();
            ck(cudaMalloc(&p, bytes), "cudaMalloc");
        }
        if (bytes >= kMinBytes && !off) {
            std::lock_guard<std::mutex> lk(mu_);
            live_[p] = bytes;
        }
        return p;
    }
    void put(int dev, void* p) {
        size_t bytes = 0;
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto it = live_.find(p);
            if (it != live_.end()) {
                bytes = it->second;
                live_.erase(it);
            }
        }
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        cudaDeviceSynchronize();  // cudaFree semantics: no pending kernel still uses the block
        if (cur != dev && cur >= 0) cudaSetDevice(cur);
        if (!bytes) {
            cudaFree(p);
            return;
        }
        std::lock_guard<std::mutex> lk(mu_);
        blocks_.push_back({dev, bytes, p});
        held_ += bytes;
        while (held_ > kCacheBytes && !blocks_.empty()) {  // oldest first
            held_ -= blocks_.front().bytes;
            cudaFree(blocks_.front().p);
            blocks_.erase(blocks_.begin());
        }
    }
    void trim() {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto& b : blocks_) {
            int cur = -1;
            cudaGetDevice(&cur);
            cudaSetDevice(b.dev);
            cudaFree(b.p);
            cudaSetDevice(cur);
        }
        blocks_.clear();
        held_ = 0;
    }

  private:
    struct Block {
        int dev;
        size_t bytes;
        void* p;
    };
    std::mutex mu_;
    std::vector<Block> blocks_;
    std::unordered_map<void*, size_t> live_;
    size_t held_ = 0;
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache;  // never destroyed: frees at process exit are the driver's
    return *c;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    int dev = 0;
    void alloc(size_t count) {
        release();
        n = count;
        if (count) {
            ck(cudaGetDevice(&dev), "cudaGetDevice");
            p = static_cast<T*>(block_cache().get(dev, count * sizeof(T)));
        }
    }
    void release() {
        if (p) block_cache().put(dev, p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
};

uint64_t align_up(uint64_t n, uint64_t a) { return (n + a - 1) / a * a; }

// MACKO_TIMING=1: host wall time of setup phases (compressor, plan) on stderr.
struct PhaseTimer {
    bool on = std::getenv("MACKO_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[macko timing] %-28s %8.3f ms (total %8.3f ms)\n", what,
                     std::chrono::duration<double, std::milli>(now - last).count(),
                     std::chrono::duration<double, std::milli>(now - t0).count());
        last = now;
    }
};
uint64_t values_bytes(uint64_t pad_nnz) { return align_up(pad_nnz * 2, 16); }
uint64_t delta_bytes(uint64_t pad_nnz, unsigned bits) { return align_up((pad_nnz * bits + 7) / 8, 16); }


}  // namespace

// Per-stream mutable state of one matrix (a handle is read-only after build and
// may be shared across streams and threads).  SpMVs on one stream are ordered, so everything a
// launch writes besides y lives here: the split-row arrival counters (zero between launches:
// each launch's last arrival resets them) and partial sums, the aligned copy of a misaligned x,
// and macko_spmv_host's device x / y.  A captured CUDA graph keeps the workspace of its capture
// stream.
struct Workspace {
    DevBuf<uint32_t> counters;  // n_split arrival counters
    DevBuf<float> partials;     // n_slots x kMaxBatch per-unit partial sums of split rows
    DevBuf<uint16_t> xcopy;     // texture-aligned copy of a misaligned x
    DevBuf<uint16_t> hx, hy;    // macko_spmv_host device buffers (hx texture-aligned inside)
    uint16_t* hx_aligned = nullptr;
    DevBuf<uint16_t> xt;        // SpMM: interleaved X (cols x 8 fp16, texture-aligned inside)
    uint16_t* xt_aligned = nullptr;
    cudaTextureObject_t xt_tex[3] = {0, 0, 0};  // over xt with 4 / 8 / 16-byte texels (kb 2 / 4 / 8)
    ~Workspace() {
        for (auto t : xt_tex)
            if (t) cudaDestroyTextureObject(t);
    }
};

constexpr size_t kMaxWorkspaces = 16;  // streams per matrix before the pool is recycled
constexpr size_t kMaxTextures = 64;    // cached x texture objects per matrix

struct macko_dev_matrix {
    int device = 0;
    int sms = 0;
    uint64_t rows = 0, cols = 0, pad_nnz = 0;
    uint32_t b_delta = 4;
    DevBuf<uint16_t> values;
    DevBuf<uint8_t> deltas;
    DevBuf<uint32_t> row_ptrs;
    std::vector<uint32_t> h_row_ptrs;
    // SpMV plan (immutable between macko_dev_configure calls)
    int x_mode = 1;             // 0 texture only, 1 fp16 smem table, 6 / 7 / 8 / 10 table + texture split
    int force_x_mode = -1;      // macko_dev_configure override (-1 = automatic rule)
    int force_ctas = 0;
    uint32_t ring = 0;          // TMA ring slots per warp
    size_t ring_offset = 0;     // x table bytes (rings follow it in dynamic smem)
    size_t smem = 0;
    size_t smem_budget = 0, per_slot = 0;  // dynamic smem left for x table + rings; bytes of one ring slot
    int grid = 0, ctas_per_sm = 0;
    uint32_t warps_active = mk::kSpmvWarpsPerCta;  // warps per CTA with a plan record
    uint32_t plan_skew = 0;                        // PlanGrid::R for K = 65536 (macko_dev_set_chain_skew)
    uint32_t n_chunks = 0, n_split = 0;
    uint64_t n_units = 0, n_slots = 0;
    DevBuf<uint32_t> plan_recs;  // W mk::WarpPlan records
    DevBuf<uint32_t> plan_u32;   // S split records {slot, first, pieces, 0}
    mk::SpmvPlanDev plan{};      // counters / partials filled per launch from the stream's workspace
    mk::PeerTable h_peers{};  // fused all-gather destinations (macko_dev_set_peers), passed per launch
    uint32_t n_peer = 0;
    int tex_align = 0;
    // per-stream workspaces and the x texture cache (guarded by mu)
    mutable std::mutex mu;
    mutable std::vector<std::unique_ptr<Workspace>> ws_pool;
    mutable std::map<cudaStream_t, Workspace*> ws_of;
    mutable std::map<const void*, cudaTextureObject_t> tex_of;
    void drop_textures() const {
        for (auto& kv : tex_of) cudaDestroyTextureObject(kv.second);
        tex_of.clear();
    }
    ~macko_dev_matrix() { drop_textures(); }
};

namespace {

int sm_count(int dev) {
    int n = 0;
    ck(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    return n;
}

void check_bits(uint32_t bits) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8))
        fail(MACKO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits; got " + std::to_string(bits));
}

void release_workspaces(macko_dev_matrix* m) {
    // a re-plan changes the workspace sizes: no launch of the old plan may still be running
    if (!m->ws_pool.empty()) {
        ck(cudaDeviceSynchronize(), "re-plan sync");
        m->ws_of.clear();
        m->ws_pool.clear();
    }
}

mk::PlanGrid plan_grid(const macko_dev_matrix* m) {
    return mk::PlanGrid{(uint32_t)m->grid, m->warps_active, 65536u, m->plan_skew};
}

// The plan's reference implementation on the host (MACKO_HOST_PLAN=1; tests compare it with the
// device builder, plan.cu, record for record).
void build_plan_host(macko_dev_matrix* m, cudaStream_t st, uint32_t W) {
    using namespace mk;
    PhaseTimer tm;
    if (m->h_row_ptrs.size() != m->rows + 1) {
        m->h_row_ptrs.resize(m->rows + 1);
        ck(cudaMemcpyAsync(m->h_row_ptrs.data(), m->row_ptrs.p, (m->rows + 1) * 4, cudaMemcpyDeviceToHost, st),
           "readback");
        ck(cudaStreamSynchronize(st), "sync");
    }
    const uint64_t R = m->rows;
    const std::vector<uint32_t>& rp = m->h_row_ptrs;

    auto row_geom = [&](uint64_t r, uint64_t& T, uint64_t& n_r) {
        const uint64_t s = rp[r], e = rp[r + 1], al = s & ~7ull;
        T = e > s ? (e - al + kStepElts - 1) / kStepElts : 0;
        n_r = T >= (uint64_t)kUnitSteps ? T / kUnitSteps : 1;  // the last unit absorbs a short remainder
    };
    auto unit_end_step = [&](uint64_t T, uint64_t n_r, uint64_t j) { return j + 1 == n_r ? T : (j + 1) * kUnitSteps; };
    const uint64_t row_w = plan_row_weight();
    auto unit_weight = [&](uint64_t T, uint64_t n_r, uint64_t j) {
        const uint64_t steps = unit_end_step(T, n_r, j) - std::min<uint64_t>(T, j * kUnitSteps);
        return steps * kStepElts + (j == 0 ? row_w : 0);
    };
    uint64_t total_w = 0, U = 0;
    for (uint64_t r = 0; r < R; ++r) {
        uint64_t T, n_r;
        row_geom(r, T, n_r);
        for (uint64_t j = 0; j < n_r; ++j) total_w += unit_weight(T, n_r, j);
        U += n_r;
    }
    m->n_units = U;
    if (U >= 0xFFFFFFFFull) fail(MACKO_EINVAL, "matrix too large for the u32 unit plan");
    std::vector<uint32_t> chunk_unit(W + 1, (uint32_t)U), chunk_row(W, 0), chunk_j(W, 0);
    std::vector<uint32_t> chunk_e(2 * (size_t)W, 0);  // [first, end) element streamed by TMA
    std::vector<int32_t> chunk_sid(2 * (size_t)W, -1);
    const uint64_t pad_nnz = rp[R];
    std::vector<uint32_t> split_slot, split_first, split_pieces;
    uint64_t slots = 0;
    int64_t prev_k = -1;
    uint64_t cw = 0, u = 0;
    for (uint64_t r = 0; r < R; ++r) {
        uint64_t T, n_r;
        row_geom(r, T, n_r);
        int64_t kf = -1, kl = -1;
        uint64_t first_units = 0, pieces = 0;
        for (uint64_t j = 0; j < n_r; ++j, ++u) {
            const uint64_t w = unit_weight(T, n_r, j);
            const uint64_t mid2 = 2 * cw + w;  // twice the unit midpoint
            int64_t k = (int64_t)plan_warp_of(mid2, 2 * (unsigned __int128)std::max<uint64_t>(total_w, 1), plan_grid(m));
            if (k < prev_k) k = prev_k;
            for (int64_t q = prev_k + 1; q <= k; ++q) {
                chunk_unit[q] = (uint32_t)u;
                chunk_row[q] = (uint32_t)r;
                chunk_j[q] = (uint32_t)j;
            }
            prev_k = k;
            if (T) {  // element range of the unit's steps, clamped to the payload
                const uint64_t al = rp[r] & ~7ull;
                const uint32_t lo = (uint32_t)(al + j * kUnitElts);
                const uint32_t hi = (uint32_t)std::min<uint64_t>(al + kStepElts * unit_end_step(T, n_r, j), pad_nnz);
                if (chunk_e[2 * k + 1] == 0) chunk_e[2 * k] = lo;
                chunk_e[2 * k + 1] = std::max(chunk_e[2 * k + 1], hi);
            }
            if (j == 0) kf = k;
            if (k == kf) ++first_units;
            if (j == 0 || k != kl) ++pieces;  // distinct (non-empty) chunks touching the row
            kl = k;
            cw += w;
        }
        if (kf != kl) {
            const int32_t sid = (int32_t)split_slot.size();
            split_slot.push_back((uint32_t)slots);
            split_first.push_back((uint32_t)first_units);
            split_pieces.push_back((uint32_t)pieces);
            slots += n_r;
            chunk_sid[2 * kf + 1] = sid;
            if (chunk_row[kf] == r && chunk_j[kf] == 0) chunk_sid[2 * kf] = sid;
            for (int64_t k = kf + 1; k <= kl; ++k) {
                chunk_sid[2 * k] = sid;
                if (k < kl) chunk_sid[2 * k + 1] = sid;
            }
        }
    }
    const uint32_t S = (uint32_t)split_slot.size();
    m->n_split = S;
    tm.mark("plan: host unit walk");
    // upload: one 48-byte record per warp, one 16-byte record per split row, counters
    std::vector<mk::WarpPlan> recs(W);
    for (uint32_t k = 0; k < W; ++k) {
        mk::WarpPlan& c = recs[k];
        c.units_left = chunk_unit[k + 1] - chunk_unit[k];
        c.row = chunk_row[k];
        c.j = chunk_j[k];
        c.e0 = chunk_e[2 * (size_t)k];
        c.e1 = chunk_e[2 * (size_t)k + 1];
        c.s = c.units_left ? rp[c.row] : 0;
        c.e = c.units_left ? rp[c.row + 1] : 0;
        c.colbase = -1;  // plan_colbase_kernel
        c.sid0 = chunk_sid[2 * (size_t)k];
        c.sid1 = chunk_sid[2 * (size_t)k + 1];
        c.slot0 = c.sid0 >= 0 ? split_slot[c.sid0] : 0;
        c.slot1 = c.sid1 >= 0 ? split_slot[c.sid1] : 0;
    }
    std::vector<uint32_t> sp(4 * (size_t)std::max<uint32_t>(S, 1), 0);  // split records
    for (uint32_t q = 0; q < S; ++q) {
        sp[4 * (size_t)q] = split_slot[q];
        sp[4 * (size_t)q + 1] = split_first[q];
        sp[4 * (size_t)q + 2] = split_pieces[q];
    }
    m->n_slots = slots;
    release_workspaces(m);
    m->plan_recs.alloc(recs.size() * sizeof(mk::WarpPlan) / 4);
    m->plan_u32.alloc(sp.size());
    ck(cudaMemcpyAsync(m->plan_recs.p, recs.data(), recs.size() * sizeof(mk::WarpPlan), cudaMemcpyHostToDevice, st),
       "plan upload");
    ck(cudaMemcpyAsync(m->plan_u32.p, sp.data(), sp.size() * 4, cudaMemcpyHostToDevice, st), "plan upload");
    mk::SpmvPlanDev& P = m->plan;
    P.warps = reinterpret_cast<const mk::WarpPlan*>(m->plan_recs.p);
    P.splits = reinterpret_cast<const uint4*>(m->plan_u32.p);
    P.counters = nullptr;
    P.partials = nullptr;
    ck(launch_plan_colbase(m->deltas.p, m->b_delta, reinterpret_cast<mk::WarpPlan*>(m->plan_recs.p), W, st),
       "plan colbase");
    g_launches.fetch_add(1);
    ck(cudaStreamSynchronize(st), "plan sync");  // host vectors go out of scope
    tm.mark("plan (host): upload + colbase + sync");
}

// The plan built on the device (plan.cu): one readback of the totals.
void build_plan_device(macko_dev_matrix* m, cudaStream_t st, uint32_t W) {
    using namespace mk;
    const uint64_t R = m->rows, ub = plan_unit_bound(R, m->pad_nnz);
    if (ub >= 0xFFFFFFFFull) fail(MACKO_EINVAL, "matrix too large for the u32 unit plan");
    DevBuf<uint32_t> u32buf;
    DevBuf<unsigned long long> u64buf;
    // u32 scratch: nu R | uo R+1 | ku, urow, uj ub | chunk_unit W+1, chunk_row W, chunk_j W | chunk_sid 2W |
    //              is_split, split_units, first_units, pieces R | sid_of, slot_of R+1
    const uint64_t n32 = R + (R + 1) + 3 * ub + (W + 1) + 2 * (uint64_t)W + 2 * (uint64_t)W + 4 * R + 2 * (R + 1);
    u32buf.alloc(n32);
    u64buf.alloc(R + (R + 1) + 2);  // rw | cw | PlanTotals (16 bytes)
    PlanTemp t{};
    uint32_t* q = u32buf.p;
    auto take = [&](uint64_t n) { uint32_t* p = q; q += n; return p; };
    t.nu = take(R);
    t.uo = take(R + 1);
    t.ku = take(ub);
    t.urow = take(ub);
    t.uj = take(ub);
    t.chunk_unit = take(W + 1);
    t.chunk_row = take(W);
    t.chunk_j = take(W);
    t.chunk_sid = reinterpret_cast<int32_t*>(take(2 * (uint64_t)W));
    t.is_split = take(R);
    t.split_units = take(R);
    t.first_units = take(R);
    t.pieces = take(R);
    t.sid_of = take(R + 1);
    t.slot_of = take(R + 1);
    t.rw = u64buf.p;
    t.cw = u64buf.p + R;
    PlanTotals* d_tot = reinterpret_cast<PlanTotals*>(u64buf.p + R + (R + 1));  // 16 bytes: 2 u64 slots
    release_workspaces(m);
    m->plan_recs.alloc((uint64_t)W * sizeof(WarpPlan) / 4);
    m->plan_u32.alloc(4 * (uint64_t)std::max<uint32_t>(W, 1));
    ck(plan_build_device(m->row_ptrs.p, (uint32_t)R, (uint32_t)m->pad_nnz, plan_grid(m), ub, m->sms, plan_row_weight(), t,
                         reinterpret_cast<WarpPlan*>(m->plan_recs.p), reinterpret_cast<uint4*>(m->plan_u32.p), d_tot, st),
       "plan build");
    ck(launch_plan_colbase(m->deltas.p, m->b_delta, reinterpret_cast<WarpPlan*>(m->plan_recs.p), W, st), "plan colbase");
    g_launches.fetch_add(13);
    PlanTotals h{};
    ck(cudaMemcpyAsync(&h, d_tot, sizeof h, cudaMemcpyDeviceToHost, st), "plan totals");
    ck(cudaStreamSynchronize(st), "plan sync");  // scratch goes out of scope
    m->n_units = h.units;
    m->n_split = h.splits;
    m->n_slots = h.slots;
    SpmvPlanDev& P = m->plan;
    P.warps = reinterpret_cast<const WarpPlan*>(m->plan_recs.p);
    P.splits = reinterpret_cast<const uint4*>(m->plan_u32.p);
    P.counters = nullptr;
    P.partials = nullptr;
}

// Warps per CTA that get a plan record (MACKO_ACTIVE_WARPS overrides, experiments).
uint32_t choose_active_warps(const macko_dev_matrix* m) {
    if (const char* e = std::getenv("MACKO_ACTIVE_WARPS")) {
        const int v = std::atoi(e);
        if (v >= 1 && v <= mk::kSpmvWarpsPerCta) return (uint32_t)v;
    }
    (void)m;
    return mk::kSpmvWarpsPerCta;
}

// Static plan: cut the unit stream into `W` equal-weight chunks (one per warp), see spmv.cuh.
void build_plan(macko_dev_matrix* m, cudaStream_t st) {
    using namespace mk;
    PhaseTimer tm;
    // Shared memory: fp16 x table with zero guards (every x_mode but 0) + per-warp TMA rings.
    int optin = 0, per_sm = 0;
    ck(cudaDeviceGetAttribute(&m->tex_align, cudaDevAttrTextureAlignment, m->device), "texture alignment");
    ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device), "smem attribute");
    ck(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, m->device), "smem attribute");
    // kSpmvCtasPerSm CTAs must fit one SM (1 KiB per CTA is reserved by the system; static smem:
    // the mbarriers and the fused all-gather stash)
    const size_t per_cta = std::min<size_t>((size_t)optin, (size_t)per_sm / kSpmvCtasPerSm - 1024);
    const size_t static_smem = spmv_static_smem();
    if (static_smem == 0) fail(MACKO_ECUDA, "SpMV kernel attributes");
    const size_t budget = per_cta - static_smem;
    const size_t per_slot = (size_t)kSpmvWarpsPerCta * (kChunkVBytes + kChunk * m->b_delta / 8);
    auto x_bytes = [&](int mode) -> size_t {
        return mode == 0 ? 0 : align_up(2 * (m->cols + mk::kXGuardLo + mk::kXGuardHi), 128);
    };
    auto ring_for = [&](int mode) -> uint32_t {
        const size_t xb = x_bytes(mode);
        if (xb >= budget) return 0;
        return kMaxRing * per_slot <= budget - xb ? kMaxRing : 0u;  // the kernel's compile-time ring
    };
    if (m->force_x_mode >= 0) {
        m->x_mode = m->force_x_mode;
    } else {
        // TEX gathers cost ~1 wavefront per 128-B line a warp gather touches, which grows with the
        // column spread of a step (~256/d columns); LDS gathers cost ~3.3 bank wavefronts at any
        // density.  Measured best split (profiles/r01_x_mode_sweep.md, re-measured in
        // profiles/r02_experiments.md after the IDP.4A addressing, 36864x12288): 4 / 3 of 8 slots
        // by TEX alternating between the two steps of a pair at d >= 0.45, 3 at 0.25 <= d < 0.45,
        // 2 below.
        // At low density the texture gathers need x resident in L1: the unified 256 KB L1/shared
        // memory keeps what the x table and the rings leave (C = 32768: ~28 KB < 64 KB of x), so
        // there the shared table alone is faster (131072x32768 @90 %: 51 vs 78 us per 16k-row slab).
        const double d = (double)m->pad_nnz / ((double)m->rows * (double)m->cols);
        const size_t smem_all = x_bytes(6) + (size_t)ring_for(6) * per_slot;
        const bool x_in_l1 = (size_t)per_sm + 24 * 1024 >= smem_all + 2 * m->cols + 16 * 1024;
        const int split = d >= 0.45 ? 10 : d >= 0.25 ? 6 : x_in_l1 ? 8 : 1;
        m->x_mode = ring_for(split) >= 2 ? split : 0;
    }
    m->smem_budget = budget;
    m->per_slot = per_slot;
    m->ring = ring_for(m->x_mode);
    if (m->ring < 2) fail(MACKO_EINVAL, "x staging mode does not leave room for the TMA rings");
    m->ring_offset = x_bytes(m->x_mode);
    m->smem = m->ring_offset + m->ring * per_slot;
    ck(spmv_occupancy(m->x_mode, (int)m->b_delta, m->smem, &m->ctas_per_sm), "spmv occupancy");
    if (m->ctas_per_sm < 1) fail(MACKO_ECUDA, "SpMV kernel cannot be resident (shared memory / registers)");
    if (m->ctas_per_sm < kSpmvCtasPerSm) fail(MACKO_ECUDA, "SpMV CTAs do not fit kSpmvCtasPerSm per SM");
    m->ctas_per_sm = kSpmvCtasPerSm;  // persistent: 32 warps per SM
    m->grid = m->sms * m->ctas_per_sm;
    // macko_dev_configure(ctas_per_sm = k > 0): use k/4 of the CTAs (a different plan, same y)
    if (m->force_ctas > 0) m->grid = std::max(1, std::min(m->grid, m->grid * m->force_ctas / 4));
    m->warps_active = choose_active_warps(m);
    const uint32_t W = (uint32_t)m->grid * m->warps_active;
    m->n_chunks = W;
    // element indices are u32 in the kernel and the ring reads up to one chunk past pad_nnz
    if (m->pad_nnz > 0xFFFFFFFFull - 2 * kChunk) fail(MACKO_EINVAL, "pad_nnz within two chunks of 2^32: no SpMV plan");
    if (std::getenv("MACKO_HOST_PLAN"))
        build_plan_host(m, st, W);
    else
        build_plan_device(m, st, W);
    tm.mark("plan");
}

void device_validate(macko_dev_matrix* m, cudaStream_t st) {
    DevBuf<uint32_t> err;
    err.alloc(1);
    ck(cudaMemsetAsync(err.p, 0, 4, st), "memset");
    ck(mk::launch_validate(m->values.p, m->deltas.p, m->row_ptrs.p, (uint32_t)m->rows, (uint32_t)m->cols, m->b_delta,
                           err.p, m->sms, st),
       "validate");
    g_launches.fetch_add(1);
    uint32_t h = 0;
    ck(cudaMemcpyAsync(&h, err.p, 4, cudaMemcpyDeviceToHost, st), "validate readback");
    ck(cudaStreamSynchronize(st), "validate sync");
    if (h & 4u) fail(MACKO_EFORMAT, "row_pointers not monotone");
    if (h & 1u) fail(MACKO_EFORMAT, "decoded column index past the column bound");
    if (h & 2u) fail(MACKO_EFORMAT, "padding value must be +0");
}

bool stream_capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return cs != cudaStreamCaptureStatusNone;
}

// The stream's workspace (caller holds m->mu).  Workspaces are allocated and zeroed outside any
// stream capture (the first SpMV on a stream, or warm-up before capturing); when the pool is full
// and no stream captures, the device is synchronised and the pool is reassigned.
Workspace* workspace(const macko_dev_matrix* m, cudaStream_t st) {
    auto it = m->ws_of.find(st);
    if (it != m->ws_of.end()) return it->second;
    if (stream_capturing(st))
        fail(MACKO_EINVAL, "first SpMV of this matrix on a capturing stream: run it once on that stream before capture");
    if (m->ws_pool.size() >= kMaxWorkspaces) {
        ck(cudaDeviceSynchronize(), "workspace recycle");
        m->ws_of.clear();
        m->ws_pool.clear();
    }
    auto w = std::make_unique<Workspace>();
    w->counters.alloc(std::max<uint32_t>(m->n_split, 1));
    w->partials.alloc(std::max<uint64_t>(m->n_slots, 1) * mk::kMaxBatch);
    ck(cudaMemsetAsync(w->counters.p, 0, w->counters.n * 4, st), "workspace zero");
    Workspace* raw = w.get();
    m->ws_pool.push_back(std::move(w));
    m->ws_of[st] = raw;
    return raw;
}

// x as the kernel reads it: 16-byte aligned for the shared-memory staging and texture-aligned
// for the TEX gathers; a misaligned x is first copied into the stream's aligned scratch buffer.
// Texture objects are cached per x buffer and destroyed only with the matrix (or when the cache
// is recycled after a device synchronisation), never while a launch may still read them.
const uint16_t* x_view(const macko_dev_matrix* m, Workspace* w, const uint16_t* d_x, bool need_tex,
                       cudaTextureObject_t* tex, cudaStream_t st) {
    const uintptr_t align = std::max<uintptr_t>(16, (uintptr_t)m->tex_align);
    if (reinterpret_cast<uintptr_t>(d_x) % align != 0) {
        if (!w->xcopy.p) {
            if (stream_capturing(st)) fail(MACKO_EINVAL, "misaligned x first seen during stream capture");
            w->xcopy.alloc(m->cols);
        }
        ck(cudaMemcpyAsync(w->xcopy.p, d_x, m->cols * 2, cudaMemcpyDeviceToDevice, st), "x copy");
        d_x = w->xcopy.p;
    }
    *tex = 0;
    if (!need_tex) return d_x;
    auto it = m->tex_of.find(d_x);
    if (it != m->tex_of.end()) {
        *tex = it->second;
        return d_x;
    }
    if (m->tex_of.size() >= kMaxTextures) {
        if (stream_capturing(st)) fail(MACKO_EINVAL, "x texture cache full during stream capture");
        ck(cudaDeviceSynchronize(), "texture cache recycle");
        m->drop_textures();
    }
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<uint16_t*>(d_x);
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned short>();
    rd.res.linear.sizeInBytes = m->cols * 2;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t = 0;
    ck(cudaCreateTextureObject(&t, &rd, &td, nullptr), "x texture");
    m->tex_of[d_x] = t;
    *tex = t;
    return d_x;
}

// ------------------------------------------------------------------------------------------
// MCKO container (io.cpp absent): 32-byte little-endian header
//   "MCKO" | u16 version = 1 | u8 b_val = 16 | u8 b_delta | u64 R | u64 C | u64 pad_nnz
// then row_pointers ((R+1) x u32 LE), packed_deltas (macko_delta_bytes), values (u16 LE,
// macko_values_bytes) back to back.  Readers reject a bad magic / version / truncated section
// (MACKO_EIO = IoError) and any invariant violation after decode (MACKO_EFORMAT = FormatError).
// ------------------------------------------------------------------------------------------
constexpr size_t kMckoHeader = 32;

struct MckoHeader {
    uint32_t b_delta = 4;
    uint64_t rows = 0, cols = 0, pad_nnz = 0;
};

void put_u16(uint8_t* p, uint16_t v) {
    p[0] = (uint8_t)v;
    p[1] = (uint8_t)(v >> 8);
}
void put_u64(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint16_t get_u16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}
bool host_little_endian() {
    const uint16_t one = 1;
    return *reinterpret_cast<const uint8_t*>(&one) == 1;
}

struct File {
    FILE* f = nullptr;
    File(const char* path, const char* mode) {
        if (!path) fail(MACKO_EINVAL, "null path");
        f = std::fopen(path, mode);
        if (!f) fail(MACKO_EIO, std::string("cannot open ") + path);
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void write(const void* p, size_t n) {
        if (n && std::fwrite(p, 1, n, f) != n) fail(MACKO_EIO, "short write");
    }
    void read(void* p, size_t n, const char* what) {
        if (n && std::fread(p, 1, n, f) != n) fail(MACKO_EIO, std::string("truncated ") + what + " section");
    }
    void zeros(size_t n) {
        static const uint8_t z[16] = {0};
        while (n) {
            const size_t k = std::min<size_t>(n, 16);
            write(z, k);
            n -= k;
        }
    }
};

void write_header(File& f, const MckoHeader& h) {
    uint8_t b[kMckoHeader] = {'M', 'C', 'K', 'O'};
    put_u16(b + 4, 1);
    b[6] = 16;
    b[7] = (uint8_t)h.b_delta;
    put_u64(b + 8, h.rows);
    put_u64(b + 16, h.cols);
    put_u64(b + 24, h.pad_nnz);
    f.write(b, sizeof b);
}

MckoHeader read_header(File& f) {
    uint8_t b[kMckoHeader];
    f.read(b, sizeof b, "header");
    if (std::memcmp(b, "MCKO", 4) != 0) fail(MACKO_EIO, "bad magic (not an MCKO file)");
    if (get_u16(b + 4) != 1) fail(MACKO_EIO, "unsupported MCKO version " + std::to_string(get_u16(b + 4)));
    if (b[6] != 16) fail(MACKO_EFORMAT, "value width must be 16 bits");
    MckoHeader h;
    h.b_delta = b[7];
    h.rows = get_u64(b + 8);
    h.cols = get_u64(b + 16);
    h.pad_nnz = get_u64(b + 24);
    if (!(h.b_delta == 1 || h.b_delta == 2 || h.b_delta == 4 || h.b_delta == 8))
        fail(MACKO_EFORMAT, "delta width must be one of 1, 2, 4, 8 bits; got " + std::to_string(h.b_delta));
    if (h.rows == 0 || h.cols == 0 || h.rows >= 0x7FFFFFFFull || h.cols >= 0x7FFFFFFFull)
        fail(MACKO_EFORMAT, "matrix dimensions out of range");
    if (h.pad_nnz > 0xFFFFFFFFull) fail(MACKO_EFORMAT, "pad_nnz does not fit u32 row pointers (SPEC.md:403)");
    return h;
}

// Row pointers section: read + check (row_pointers[0] = 0, monotone, row_pointers[R] = pad_nnz).
std::vector<uint32_t> read_row_ptrs(File& f, const MckoHeader& h) {
    std::vector<uint32_t> rp(h.rows + 1);
    std::vector<uint8_t> raw((h.rows + 1) * 4);
    f.read(raw.data(), raw.size(), "row_pointers");
    for (uint64_t i = 0; i <= h.rows; ++i)
        rp[i] = raw[4 * i] | (raw[4 * i + 1] << 8) | (raw[4 * i + 2] << 16) | ((uint32_t)raw[4 * i + 3] << 24);
    if (rp[0] != 0) fail(MACKO_EFORMAT, "row_pointers[0] must be 0");
    for (uint64_t r = 0; r < h.rows; ++r)
        if (rp[r + 1] < rp[r]) fail(MACKO_EFORMAT, "row_pointers not monotone");
    if (rp[h.rows] != h.pad_nnz) fail(MACKO_EFORMAT, "row_pointers[R] != pad_nnz in the header");
    return rp;
}

// validate_macko (convert.hpp:25-27) on host arrays: codewords decode to strictly increasing
// columns < C, padding entries (codeword all-ones followed by... any entry with value +/-0) are +0.
void host_validate(const MckoHeader& h, const std::vector<uint32_t>& rp, const uint8_t* deltas, const uint16_t* values) {
    const uint32_t bits = h.b_delta, per = 8 / bits, mask = (1u << bits) - 1u;
    for (uint64_t r = 0; r < h.rows; ++r) {
        int64_t col = -1;
        for (uint64_t e = rp[r]; e < rp[r + 1]; ++e) {
            col += ((deltas[e / per] >> ((e % per) * bits)) & mask) + 1;
            if ((uint64_t)col >= h.cols) fail(MACKO_EFORMAT, "decoded column index past the column bound");
            if ((values[e] & 0x7FFFu) == 0 && values[e] != 0) fail(MACKO_EFORMAT, "padding value must be +0");
        }
    }
}

// Streams `bytes` from the file into device memory through two pinned staging buffers, so the
// disk read of one block overlaps the H2D copy of the previous one.
void stream_to_device(File& f, void* dst, uint64_t bytes, cudaStream_t st, const char* what) {
    constexpr size_t kBlock = 32u << 20;
    uint8_t* pinned[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    struct Cleanup {
        uint8_t** p;
        cudaEvent_t* e;
        ~Cleanup() {
            for (int i = 0; i < 2; ++i) {
                if (e[i]) {
                    cudaEventSynchronize(e[i]);
                    cudaEventDestroy(e[i]);
                }
                if (p[i]) cudaFreeHost(p[i]);
            }
        }
    } cleanup{pinned, done};
    const size_t blk = (size_t)std::min<uint64_t>(bytes, kBlock);
    if (!blk) return;
    for (int i = 0; i < 2; ++i) {
        ck(cudaMallocHost(&pinned[i], blk), "pinned staging buffer");
        ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "event");
    }
    bool used[2] = {false, false};
    uint64_t off = 0;
    for (int i = 0; off < bytes; i ^= 1) {
        const size_t n = (size_t)std::min<uint64_t>(bytes - off, blk);
        if (used[i]) ck(cudaEventSynchronize(done[i]), "staging wait");
        f.read(pinned[i], n, what);
        ck(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, pinned[i], n, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaEventRecord(done[i], st), "event");
        used[i] = true;
        off += n;
    }
}

// Matrix Market coordinate real/integer general -> dense fp16 (row-major), entries converted
// like the reference's float_to_half (fp16.cpp:37-73: RNE) from the parsed value.
void read_mm(const char* path, uint64_t* rows, uint64_t* cols, uint16_t* dense) {
    File f(path, "r");
    char line[4096];
    if (!std::fgets(line, sizeof line, f.f)) fail(MACKO_EIO, "empty Matrix Market file");
    std::string hdr(line);
    for (auto& c : hdr) c = (char)std::tolower((unsigned char)c);
    if (hdr.rfind("%%matrixmarket", 0) != 0) fail(MACKO_EIO, "missing %%MatrixMarket banner");
    if (hdr.find("matrix") == std::string::npos || hdr.find("coordinate") == std::string::npos ||
        (hdr.find("real") == std::string::npos && hdr.find("integer") == std::string::npos) ||
        hdr.find("general") == std::string::npos)
        fail(MACKO_EIO, "unsupported Matrix Market kind (need: matrix coordinate real|integer general)");
    unsigned long long R = 0, C = 0, nnz = 0;
    for (;;) {
        if (!std::fgets(line, sizeof line, f.f)) fail(MACKO_EIO, "missing size line");
        if (line[0] == '%' || line[strspn(line, " \t\r\n")] == 0) continue;
        if (std::sscanf(line, "%llu %llu %llu", &R, &C, &nnz) != 3) fail(MACKO_EIO, "bad size line");
        break;
    }
    if (R == 0 || C == 0 || R >= 0x7FFFFFFFull || C >= 0x7FFFFFFFull) fail(MACKO_EFORMAT, "matrix dimensions out of range");
    *rows = R;
    *cols = C;
    if (!dense) return;
    std::memset(dense, 0, R * C * 2);
    std::set<std::pair<uint64_t, uint64_t>> seen;
    for (unsigned long long k = 0; k < nnz; ++k) {
        if (!std::fgets(line, sizeof line, f.f)) fail(MACKO_EIO, "truncated Matrix Market entries");
        unsigned long long i = 0, j = 0;
        double v = 0;
        if (std::sscanf(line, "%llu %llu %lf", &i, &j, &v) != 3) fail(MACKO_EIO, "bad entry line");
        if (i < 1 || j < 1 || i > R || j > C) fail(MACKO_EFORMAT, "Matrix Market index out of range");
        if (!seen.insert({i, j}).second) fail(MACKO_EFORMAT, "duplicate Matrix Market coordinate");
        const __half hv = __float2half_rn((float)v);
        dense[(i - 1) * C + (j - 1)] = __half_as_ushort(hv);
    }
}

void check_shape(uint64_t rows, uint64_t cols) {
    if (rows == 0 || cols == 0) fail(MACKO_EINVAL, "matrix dimensions must be >= 1");
    if (rows >= 0x7FFFFFFFull || cols >= 0x7FFFFFFFull) fail(MACKO_EINVAL, "rows/cols must be < 2^31");
}

}  // namespace

extern "C" {

const char* macko_last_error(void) { return g_err.c_str(); }
uint32_t macko_unit_steps(void) { return (uint32_t)mk::kUnitSteps; }

const char* macko_version(void) { return "macko-b200 0.2 (sm_100a; SpMV and compressor for b_delta in {1,2,4,8})"; }
uint64_t macko_kernel_launches(void) { return g_launches.load(); }

uint32_t macko_density_threshold(double d) {
    if (!(d > 0)) return 0;
    if (d >= 1) return 1u << 24;
    return (uint32_t)__builtin_floor(d * 16777216.0 + 0.5);
}

macko_status macko_dev_upload(int device, uint64_t rows, uint64_t cols, uint32_t b_delta, const uint16_t* values,
                              uint64_t n_values, const uint8_t* deltas, uint64_t n_delta_bytes, const uint32_t* row_ptrs,
                              void* stream, macko_dev_matrix** out) {
    return guarded([&] {
        if (!out || !row_ptrs) fail(MACKO_EINVAL, "null argument");
        *out = nullptr;
        check_bits(b_delta);
        check_shape(rows, cols);
        if (row_ptrs[0] != 0) fail(MACKO_EFORMAT, "row_pointers[0] must be 0");
        for (uint64_t r = 0; r < rows; ++r)
            if (row_ptrs[r + 1] < row_ptrs[r]) fail(MACKO_EFORMAT, "row_pointers not monotone");
        const uint64_t pad_nnz = row_ptrs[rows];
        if (n_values < pad_nnz) fail(MACKO_EFORMAT, "values shorter than pad_nnz");
        if (n_delta_bytes * 8 < pad_nnz * b_delta) fail(MACKO_EFORMAT, "packed_deltas shorter than pad_nnz");
        if (pad_nnz && (!values || !deltas)) fail(MACKO_EINVAL, "null payload");
        DeviceGuard g(device);
        cudaStream_t st = (cudaStream_t)stream;
        auto* m = new macko_dev_matrix;
        std::unique_ptr<macko_dev_matrix> hold(m);
        m->device = device;
        m->sms = sm_count(device);
        m->rows = rows;
        m->cols = cols;
        m->pad_nnz = pad_nnz;
        m->b_delta = b_delta;
        const uint64_t vb = values_bytes(pad_nnz), db = delta_bytes(pad_nnz, b_delta);
        // one zeroed TMA chunk of slack past the payload: the SpMV's ring copies are never clamped
        m->values.alloc(vb / 2 + mk::kChunk);
        m->deltas.alloc(db + mk::kChunk);  // one chunk of codewords at up to 8 bits
        m->row_ptrs.alloc(rows + 1);
        ck(cudaMemsetAsync(m->values.p, 0, m->values.n * 2, st), "memset");
        ck(cudaMemsetAsync(m->deltas.p, 0, m->deltas.n, st), "memset");
        if (pad_nnz) {
            ck(cudaMemcpyAsync(m->values.p, values, std::min<uint64_t>(n_values * 2, vb), cudaMemcpyHostToDevice, st),
               "upload values");
            ck(cudaMemcpyAsync(m->deltas.p, deltas, std::min<uint64_t>(n_delta_bytes, db), cudaMemcpyHostToDevice, st),
               "upload deltas");
        }
        ck(cudaMemcpyAsync(m->row_ptrs.p, row_ptrs, (rows + 1) * 4, cudaMemcpyHostToDevice, st), "upload row_ptrs");
        m->h_row_ptrs.assign(row_ptrs, row_ptrs + rows + 1);
        device_validate(m, st);
        build_plan(m, st);
        *out = hold.release();
    });
}

macko_status macko_dev_from_dense(int device, const uint16_t* d_dense, uint64_t rows, uint64_t cols, uint64_t ld,
                                  uint32_t b_delta, void* stream, macko_dev_matrix** out) {
    return guarded([&] {
        if (!out || !d_dense) fail(MACKO_EINVAL, "null argument");
        *out = nullptr;
        check_bits(b_delta);
        check_shape(rows, cols);
        if (ld < cols) fail(MACKO_EINVAL, "leading dimension < cols");
        DeviceGuard g(device);
        cudaStream_t st = (cudaStream_t)stream;
        PhaseTimer tm;
        auto* m = new macko_dev_matrix;
        std::unique_ptr<macko_dev_matrix> hold(m);
        m->device = device;
        m->sms = sm_count(device);
        m->rows = rows;
        m->cols = cols;
        m->b_delta = b_delta;
        DevBuf<uint32_t> counts;
        DevBuf<int32_t> lastcol;
        DevBuf<unsigned long long> total;
        counts.alloc(rows);
        lastcol.alloc(rows);
        total.alloc(1);
        m->row_ptrs.alloc(rows + 1);
        tm.mark("scratch alloc");
        ck(mk::launch_count_rows(d_dense, ld, (uint32_t)rows, (uint32_t)cols, b_delta, counts.p, lastcol.p, m->sms, st),
           "count_rows");
        ck(mk::launch_scan_counts(counts.p, (uint32_t)rows, m->row_ptrs.p, total.p, st), "scan_counts");
        g_launches.fetch_add(2);
        unsigned long long pad_nnz = 0;
        ck(cudaMemcpyAsync(&pad_nnz, total.p, 8, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaStreamSynchronize(st), "sync");
        tm.mark("count + scan + sync");
        if (pad_nnz > 0xFFFFFFFFull) fail(MACKO_EINVAL, "pad_nnz does not fit u32 row pointers (SPEC.md:403)");
        m->pad_nnz = pad_nnz;
        const uint64_t vb = values_bytes(pad_nnz), db = delta_bytes(pad_nnz, b_delta);
        m->values.alloc(vb / 2 + mk::kChunk);  // + one zeroed TMA chunk of slack (see upload)
        m->deltas.alloc(db + mk::kChunk);  // one chunk of codewords at up to 8 bits
        ck(cudaMemsetAsync(m->deltas.p, 0, m->deltas.n, st), "memset");
        if (m->values.n * 2 > pad_nnz * 2)
            ck(cudaMemsetAsync(m->values.p + pad_nnz, 0, m->values.n * 2 - pad_nnz * 2, st), "memset");
        if (pad_nnz)
            ck(mk::launch_emit_rows(d_dense, ld, (uint32_t)rows, (uint32_t)cols, b_delta, m->row_ptrs.p, lastcol.p,
                                    m->values.p, reinterpret_cast<uint32_t*>(m->deltas.p), m->sms, st),
               "emit_rows");
        g_launches.fetch_add(1);
        tm.mark("alloc + emit launch");
        build_plan(m, st);
        tm.mark("build_plan");
        *out = hold.release();
    });
}

macko_status macko_dev_from_csr(int device, uint64_t rows, uint64_t cols, uint32_t b_delta, const uint16_t* values,
                                const uint32_t* col_idx, const uint32_t* row_ptrs, uint64_t nnz, int on_device,
                                void* stream, macko_dev_matrix** out) {
    return guarded([&] {
        if (!out || !row_ptrs || (nnz && (!values || !col_idx))) fail(MACKO_EINVAL, "null argument");
        *out = nullptr;
        check_bits(b_delta);
        check_shape(rows, cols);
        if (nnz > 0xFFFFFFFFull) fail(MACKO_EINVAL, "nnz does not fit u32 row pointers");
        DeviceGuard g(device);
        cudaStream_t st = (cudaStream_t)stream;
        DevBuf<uint32_t> drp, dci;
        DevBuf<uint16_t> dcv;
        const uint32_t* rp = row_ptrs;
        const uint32_t* ci = col_idx;
        const uint16_t* cv = values;
        if (!on_device) {  // host CsrMatrix (matrix.hpp:39-48): row pointers checked here, arrays uploaded
            if (row_ptrs[0] != 0) fail(MACKO_EINVAL, "row_pointers[0] must be 0");
            for (uint64_t r = 0; r < rows; ++r)
                if (row_ptrs[r + 1] < row_ptrs[r]) fail(MACKO_EINVAL, "row_pointers not monotone");
            if (row_ptrs[rows] != nnz) fail(MACKO_EINVAL, "row_pointers[rows] != nnz");
            drp.alloc(rows + 1);
            ck(cudaMemcpyAsync(drp.p, row_ptrs, (rows + 1) * 4, cudaMemcpyHostToDevice, st), "upload row_ptrs");
            if (nnz) {
                dci.alloc(nnz);
                dcv.alloc(nnz);
                ck(cudaMemcpyAsync(dci.p, col_idx, nnz * 4, cudaMemcpyHostToDevice, st), "upload columns");
                ck(cudaMemcpyAsync(dcv.p, values, nnz * 2, cudaMemcpyHostToDevice, st), "upload values");
            }
            rp = drp.p;
            ci = dci.p;
            cv = dcv.p;
        }
        auto* m = new macko_dev_matrix;
        std::unique_ptr<macko_dev_matrix> hold(m);
        m->device = device;
        m->sms = sm_count(device);
        m->rows = rows;
        m->cols = cols;
        m->b_delta = b_delta;
        DevBuf<uint32_t> counts, err;
        DevBuf<unsigned long long> total;
        counts.alloc(rows);
        err.alloc(1);
        total.alloc(1);
        m->row_ptrs.alloc(rows + 1);
        ck(cudaMemsetAsync(err.p, 0, 4, st), "memset");
        ck(mk::launch_csr_count(rp, ci, (uint32_t)rows, (uint32_t)cols, b_delta, counts.p, err.p, m->sms, st),
           "csr_count");
        ck(mk::launch_scan_counts(counts.p, (uint32_t)rows, m->row_ptrs.p, total.p, st), "scan_counts");
        g_launches.fetch_add(2);
        struct {
            unsigned long long total;
            uint32_t err;
        } h{};
        ck(cudaMemcpyAsync(&h.total, total.p, 8, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaMemcpyAsync(&h.err, err.p, 4, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaStreamSynchronize(st), "sync");
        // macko_from_csr rejects a non-canonical CSR
        if (h.err & 1u) fail(MACKO_EINVAL, "column index out of range");
        if (h.err & 2u) fail(MACKO_EINVAL, "columns not strictly increasing within a row");
        if (h.err & 4u) fail(MACKO_EINVAL, "row_pointers not monotone");
        if (h.total > 0xFFFFFFFFull) fail(MACKO_EINVAL, "pad_nnz does not fit u32 row pointers (SPEC.md:403)");
        const uint64_t pad_nnz = h.total;
        m->pad_nnz = pad_nnz;
        const uint64_t vb = values_bytes(pad_nnz), db = delta_bytes(pad_nnz, b_delta);
        m->values.alloc(vb / 2 + mk::kChunk);  // + one zeroed TMA chunk of slack (see upload)
        m->deltas.alloc(db + mk::kChunk);
        ck(cudaMemsetAsync(m->values.p, 0, m->values.n * 2, st), "memset");
        ck(cudaMemsetAsync(m->deltas.p, 0, m->deltas.n, st), "memset");
        if (pad_nnz) {
            DevBuf<uint8_t> codes;
            codes.alloc(pad_nnz);
            ck(mk::launch_csr_emit(rp, ci, cv, (uint32_t)rows, b_delta, m->row_ptrs.p, m->values.p, codes.p, m->sms, st),
               "csr_emit");
            ck(mk::launch_pack_codes(codes.p, pad_nnz, b_delta, m->deltas.p, (pad_nnz * b_delta + 7) / 8, m->sms, st),
               "pack_codes");
            g_launches.fetch_add(2);
            ck(cudaStreamSynchronize(st), "sync");  // codes goes out of scope
        }
        build_plan(m, st);
        *out = hold.release();
    });
}

macko_status macko_csr_from_dense(int device, const uint16_t* dense, uint64_t rows, uint64_t cols, uint64_t ld,
                                  int on_device, uint32_t* row_ptrs, uint16_t* values, uint32_t* col_idx,
                                  uint64_t* nnz, void* stream) {
    return guarded([&] {
        if (!dense || !row_ptrs || !nnz) fail(MACKO_EINVAL, "null argument");
        if (rows >= 0x7FFFFFFFull || cols >= 0x7FFFFFFFull) fail(MACKO_EINVAL, "rows/cols must be < 2^31");
        if (ld < cols) fail(MACKO_EINVAL, "leading dimension < cols");
        DeviceGuard g(device);
        cudaStream_t st = (cudaStream_t)stream;
        int sms = sm_count(device);
        DevBuf<uint16_t> dd;
        const uint16_t* d = dense;
        uint64_t dld = ld;
        if (!on_device) {
            dd.alloc(std::max<uint64_t>(rows * cols, 1));
            ck(cudaMemcpy2DAsync(dd.p, cols * 2, dense, ld * 2, cols * 2, rows, cudaMemcpyHostToDevice, st), "upload");
            d = dd.p;
            dld = cols;
        }
        DevBuf<uint32_t> counts, rp;
        DevBuf<unsigned long long> total;
        counts.alloc(std::max<uint64_t>(rows, 1));
        rp.alloc(rows + 1);
        total.alloc(1);
        ck(mk::launch_dense_nnz(d, dld, (uint32_t)rows, (uint32_t)cols, counts.p, sms, st), "dense_nnz");
        ck(mk::launch_scan_counts(counts.p, (uint32_t)rows, rp.p, total.p, st), "scan_counts");
        g_launches.fetch_add(2);
        unsigned long long n = 0;
        ck(cudaMemcpyAsync(&n, total.p, 8, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaMemcpyAsync(row_ptrs, rp.p, (rows + 1) * 4, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaStreamSynchronize(st), "sync");
        if (n > 0xFFFFFFFFull) fail(MACKO_EINVAL, "nnz does not fit u32 row pointers");
        *nnz = n;
        if (!values || !col_idx || n == 0) return;  // count-only call
        DevBuf<uint16_t> v;
        DevBuf<uint32_t> c;
        v.alloc(n);
        c.alloc(n);
        ck(mk::launch_dense_csr_emit(d, dld, (uint32_t)rows, (uint32_t)cols, rp.p, v.p, c.p, sms, st), "csr_emit");
        g_launches.fetch_add(1);
        ck(cudaMemcpyAsync(values, v.p, n * 2, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaMemcpyAsync(col_idx, c.p, n * 4, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

macko_status macko_dev_to_dense(const macko_dev_matrix* m, uint16_t* dense, uint64_t ld, int on_device, void* stream) {
    return guarded([&] {
        if (!m || !dense) fail(MACKO_EINVAL, "null argument");
        if (ld < m->cols) fail(MACKO_EINVAL, "leading dimension < cols");
        DeviceGuard g(m->device);
        cudaStream_t st = (cudaStream_t)stream;
        DevBuf<uint16_t> tmp;
        uint16_t* d = dense;
        uint64_t dld = ld;
        if (!on_device) {
            tmp.alloc(m->rows * m->cols);
            d = tmp.p;
            dld = m->cols;
        }
        ck(cudaMemset2DAsync(d, dld * 2, 0, m->cols * 2, m->rows, st), "memset");
        DevBuf<uint32_t> err;
        err.alloc(1);
        ck(cudaMemsetAsync(err.p, 0, 4, st), "memset");
        ck(mk::launch_to_dense(m->values.p, m->deltas.p, m->row_ptrs.p, (uint32_t)m->rows, (uint32_t)m->cols,
                               m->b_delta, d, dld, err.p, m->sms, st),
           "to_dense");
        g_launches.fetch_add(1);
        uint32_t h = 0;
        ck(cudaMemcpyAsync(&h, err.p, 4, cudaMemcpyDeviceToHost, st), "readback");
        if (!on_device)
            ck(cudaMemcpy2DAsync(dense, ld * 2, d, dld * 2, m->cols * 2, m->rows, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        if (h) fail(MACKO_EFORMAT, "decoded column index past the column bound");
    });
}

macko_status macko_dev_padding_count(const macko_dev_matrix* m, uint64_t* out, void* stream) {
    return guarded([&] {
        if (!m || !out) fail(MACKO_EINVAL, "null argument");
        DeviceGuard g(m->device);
        cudaStream_t st = (cudaStream_t)stream;
        DevBuf<unsigned long long> cnt;
        cnt.alloc(1);
        ck(cudaMemsetAsync(cnt.p, 0, 8, st), "memset");
        ck(mk::launch_padding_count(m->values.p, m->pad_nnz, cnt.p, m->sms, st), "padding_count");
        g_launches.fetch_add(1);
        unsigned long long h = 0;
        ck(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, st), "readback");
        ck(cudaStreamSynchronize(st), "sync");
        *out = h;
    });
}

macko_status macko_dev_get_info(const macko_dev_matrix* m, macko_dev_info* out) {
    return guarded([&] {
        if (!m || !out) fail(MACKO_EINVAL, "null argument");
        out->rows = m->rows;
        out->cols = m->cols;
        out->pad_nnz = m->pad_nnz;
        out->values_bytes = values_bytes(m->pad_nnz);
        out->delta_bytes = delta_bytes(m->pad_nnz, m->b_delta);
        out->row_ptr_bytes = 4 * (m->rows + 1);
        out->traffic_bytes = out->values_bytes + out->delta_bytes + out->row_ptr_bytes + 2 * m->cols + 2 * m->rows;
        out->b_delta = m->b_delta;
        out->device = m->device;
        out->d_values = m->values.p;
        out->d_deltas = m->deltas.p;
        out->d_row_ptrs = m->row_ptrs.p;
    });
}

macko_status macko_dev_download(const macko_dev_matrix* m, uint16_t* values, uint8_t* deltas, uint32_t* row_ptrs,
                                void* stream) {
    return guarded([&] {
        if (!m) fail(MACKO_EINVAL, "null handle");
        DeviceGuard g(m->device);
        cudaStream_t st = (cudaStream_t)stream;
        if (values)
            ck(cudaMemcpyAsync(values, m->values.p, values_bytes(m->pad_nnz), cudaMemcpyDeviceToHost, st), "download");
        if (deltas)
            ck(cudaMemcpyAsync(deltas, m->deltas.p, delta_bytes(m->pad_nnz, m->b_delta), cudaMemcpyDeviceToHost, st),
               "download");
        if (row_ptrs) ck(cudaMemcpyAsync(row_ptrs, m->row_ptrs.p, (m->rows + 1) * 4, cudaMemcpyDeviceToHost, st), "download");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

namespace {
// One SpMV launch (macko_dev_spmv_ex; macko_spmv_host adds a mapped host mirror of y).
macko_status spmv_launch(const macko_dev_matrix* m, const uint16_t* d_x, uint16_t* d_y, void* stream, uint32_t flags,
                         uint16_t* y_mirror) {
    return guarded([&] {
        if (!m || !d_x || !d_y) fail(MACKO_EINVAL, "null argument");
        if (flags & ~(uint32_t)(MACKO_SPMV_PDL | MACKO_SPMV_PEERS | MACKO_SPMV_PEER_BANK1))
            fail(MACKO_EINVAL, "unknown macko_dev_spmv_ex flag");
        if ((flags & MACKO_SPMV_PEER_BANK1) && !(flags & MACKO_SPMV_PEERS))
            fail(MACKO_EINVAL, "MACKO_SPMV_PEER_BANK1 without MACKO_SPMV_PEERS");
        if ((flags & MACKO_SPMV_PEERS) && m->n_peer == 0) fail(MACKO_EINVAL, "MACKO_SPMV_PEERS without macko_dev_set_peers");
        if (!mk::spmv_valid_config(m->x_mode, (int)m->b_delta))
            fail(MACKO_EINVAL, "no SpMV kernel for b_delta " + std::to_string(m->b_delta) + " with this x_mode");
        DeviceGuard g(m->device);
        const cudaStream_t st = (cudaStream_t)stream;
        std::lock_guard<std::mutex> lk(m->mu);
        Workspace* w = workspace(m, st);
        mk::SpmvArgs a{};
        a.values = m->values.p;
        a.deltas = m->deltas.p;
        a.row_ptrs = m->row_ptrs.p;
        const int mode = m->x_mode;
        a.x = x_view(m, w, d_x, mode != 1, &a.xtex, st);
        a.y = d_y;
        a.rows = (uint32_t)m->rows;
        a.cols = (uint32_t)m->cols;
        a.value_elems = m->values.n;
        a.delta_bytes = m->deltas.n;
        a.ring = m->ring;
        a.ring_offset = (uint32_t)m->ring_offset;
        a.warps_active = m->warps_active;
#ifdef MACKO_TRACE
        a.trace_slot = g_trace_slot.fetch_add(1);
#endif
        a.plan = m->plan;
        a.plan.counters = w->counters.p;
        a.plan.partials = w->partials.p;
        a.pdl = (flags & MACKO_SPMV_PDL) != 0;
        a.y_mirror = y_mirror;
        a.no_split = m->n_split == 0 ? 1u : 0u;
        if (flags & MACKO_SPMV_PEERS) {
            a.n_peer = m->n_peer;
            const uint32_t bank = (flags & MACKO_SPMV_PEER_BANK1) ? 1u : 0u;
            for (uint32_t p = 0; p < mk::kMaxPeers; ++p) {
                a.peer_y[p] = m->h_peers.y[bank][p];
                a.peer_flag[p] = m->h_peers.flag[p];
            }
        }
        a.value_count = (uint32_t)m->pad_nnz;
        if (m->pad_nnz == 0) {  // no stored entries: every row is empty, y = +0
            if (flags & MACKO_SPMV_PEERS) fail(MACKO_EINVAL, "fused all-gather needs stored entries");
            ck(cudaMemsetAsync(d_y, 0, m->rows * 2, st), "y = 0");
            if (y_mirror) ck(cudaMemsetAsync(y_mirror, 0, m->rows * 2, st), "y = 0");
            return;
        }
        ck(mk::launch_spmv(a, (int)m->b_delta, m->grid, mode, m->smem, st, (flags & MACKO_SPMV_PDL) != 0),
           "macko_spmv launch");
        g_launches.fetch_add(1);
    });
}
}  // namespace

macko_status macko_dev_spmv_ex(const macko_dev_matrix* m, const uint16_t* d_x, uint16_t* d_y, void* stream,
                               uint32_t flags) {
    return spmv_launch(m, d_x, d_y, stream, flags, nullptr);
}

macko_status macko_dev_spmv(const macko_dev_matrix* m, const uint16_t* d_x, uint16_t* d_y, void* stream) {
    return macko_dev_spmv_ex(m, d_x, d_y, stream, 0);
}

// SpMM gather split when the interleaved table fits beside the rings (kb = 2 up to ~28k columns;
// kb = 4 / 8 tables do not fit at 12288 columns and gather through the texture).  36864x12288
// @50 %, batch 2 (tools/spmm_time.py): x_mode 8 (2 of 8 slots by TEX) 135.0 us, 1 (table only)
// 137.6, 6 140.1, 7 178.3, 0 (texture only) 317.9.
int spmm_table_mode(uint32_t kb) { return kb == 2 ? 8 : 7; }

macko_status macko_dev_spmm(const macko_dev_matrix* m, const uint16_t* d_X, uint64_t ldx, uint16_t* d_Y, uint64_t ldy,
                            uint32_t batch, void* stream) {
    if (batch == 1) return macko_dev_spmv(m, d_X, d_Y, stream);
    return guarded([&] {
        if (!m || !d_X || !d_Y) fail(MACKO_EINVAL, "null argument");
        if (batch < 1 || batch > mk::kMaxBatch) fail(MACKO_EINVAL, "batch must be 1..8");
        if (m->b_delta != 4) fail(MACKO_EINVAL, "SpMM is built for b_delta = 4 (the paper's format)");
        if (ldx < m->cols || ldy < m->rows) fail(MACKO_EINVAL, "leading dimension smaller than the vector length");
        DeviceGuard g(m->device);
        const cudaStream_t st = (cudaStream_t)stream;
        if (m->pad_nnz == 0) {
            ck(cudaMemset2DAsync(d_Y, ldy * 2, 0, m->rows * 2, batch, st), "Y = 0");
            return;
        }
        // batch 3-4 when the 4-wide interleaved table does not fit beside the rings but the 2-wide
        // one does: two 2-wide passes (2 x 136 us) beat one 4-wide texture-only pass (357 us) at
        // 36864x12288; each column's y is the same bits either way.
        if (batch > 2 && batch <= 4 && m->b_delta == 4) {
            const size_t t4 = align_up(2 * 4 * (m->cols + mk::kXGuardLo + mk::kXGuardHi), 128);
            const size_t t2 = align_up(2 * 2 * (m->cols + mk::kXGuardLo + mk::kXGuardHi), 128);
            if (t4 + 2 * m->per_slot > m->smem_budget && t2 + 2 * m->per_slot <= m->smem_budget) {
                const macko_status s1 = macko_dev_spmm(m, d_X, ldx, d_Y, ldy, 2, stream);
                if (s1 != MACKO_OK) fail(s1, g_err);
                const macko_status s2 = macko_dev_spmm(m, d_X + 2 * ldx, ldx, d_Y + 2 * ldy, ldy, batch - 2, stream);
                if (s2 != MACKO_OK) fail(s2, g_err);
                return;
            }
        }
        const uint32_t kb = batch <= 2 ? 2u : batch <= 4 ? 4u : 8u;
        const int ti = kb == 2 ? 0 : kb == 4 ? 1 : 2;
        std::lock_guard<std::mutex> lk(m->mu);
        Workspace* w = workspace(m, st);
        const uint64_t xt_elems = m->cols * mk::kMaxBatch + 8;  // + 16 bytes: staging reads whole vectors
        if (!w->xt.p) {
            if (stream_capturing(st)) fail(MACKO_EINVAL, "first SpMM of this matrix on a capturing stream");
            const uintptr_t al = std::max<uintptr_t>(16, (uintptr_t)m->tex_align);
            w->xt.alloc(xt_elems + al / 2);
            ck(cudaMemsetAsync(w->xt.p, 0, w->xt.n * 2, st), "memset");
            const uintptr_t p = reinterpret_cast<uintptr_t>(w->xt.p);
            w->xt_aligned = reinterpret_cast<uint16_t*>((p + al - 1) / al * al);
        }
        if (!w->xt_tex[ti]) {
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeLinear;
            rd.res.linear.devPtr = w->xt_aligned;
            rd.res.linear.desc = kb == 2 ? cudaCreateChannelDesc<unsigned int>()
                                 : kb == 4 ? cudaCreateChannelDesc<uint2>() : cudaCreateChannelDesc<uint4>();
            rd.res.linear.sizeInBytes = m->cols * kb * 2;
            cudaTextureDesc td{};
            td.readMode = cudaReadModeElementType;
            ck(cudaCreateTextureObject(&w->xt_tex[ti], &rd, &td, nullptr), "XT texture");
        }
        // interleaved X, then the SpMM: x_mode 7 when the interleaved table and two ring slots fit
        // (whole 16-byte vectors: the table staging copies vectors, the tail past cols is zero)
        ck(mk::launch_interleave(d_X, ldx, batch, kb, (uint32_t)m->cols, w->xt_aligned,
                                 (uint32_t)((m->cols * kb + 7) / 8 * 8), st),
           "interleave");
        const size_t table = align_up(2 * kb * (m->cols + mk::kXGuardLo + mk::kXGuardHi), 128);
        int mode = table + 2 * m->per_slot <= m->smem_budget ? spmm_table_mode(kb) : 0;
        if (const char* e = std::getenv("MACKO_SPMM_XMODE")) {  // experiments: force a gather split
            const int f = std::atoi(e);
            if (mk::spmm_valid_x_mode(f) && (f == 0 || table + 2 * m->per_slot <= m->smem_budget)) mode = f;
        }
        mk::SpmvArgs a{};
        a.values = m->values.p;
        a.deltas = m->deltas.p;
        a.row_ptrs = m->row_ptrs.p;
        a.x = w->xt_aligned;
        a.xtex = w->xt_tex[ti];
        a.y = d_Y;
        a.ldy = ldy;
        a.batch = batch;
        a.rows = (uint32_t)m->rows;
        a.cols = (uint32_t)m->cols;
        a.value_elems = m->values.n;
        a.delta_bytes = m->deltas.n;
        a.ring = mk::kMaxRing;
        a.ring_offset = mode != 0 ? (uint32_t)table : 0u;
        a.warps_active = m->warps_active;
        a.plan = m->plan;
        a.plan.counters = w->counters.p;
        a.plan.partials = w->partials.p;
        a.value_count = (uint32_t)m->pad_nnz;
        const size_t smem = (mode != 0 ? table : 0) + mk::kMaxRing * m->per_slot;
        ck(mk::launch_spmm(a, (int)kb, m->grid, mode, smem, st), "macko_spmm launch");
        g_launches.fetch_add(2);
    });
}

macko_status macko_spmv_host(const macko_dev_matrix* m, const uint16_t* h_x, uint16_t* h_y, void* stream) {
    return guarded([&] {
        if (!m || !h_x || !h_y) fail(MACKO_EINVAL, "null argument");
        DeviceGuard g(m->device);
        cudaStream_t st = (cudaStream_t)stream;
        uint16_t *hx_dev = nullptr, *hy_dev = nullptr;
        {
            // the stream's device x / y (texture-aligned x: no staging copy inside the SpMV)
            std::lock_guard<std::mutex> lk(m->mu);
            Workspace* w = workspace(m, st);
            if (!w->hx.p) {
                const uintptr_t a = std::max<uintptr_t>(16, (uintptr_t)m->tex_align);
                w->hx.alloc(m->cols + a / 2);
                const uintptr_t p = reinterpret_cast<uintptr_t>(w->hx.p);
                w->hx_aligned = reinterpret_cast<uint16_t*>((p + a - 1) / a * a);
                w->hy.alloc(m->rows);
            }
            hx_dev = w->hx_aligned;
            hy_dev = w->hy.p;
        }
        // Pinned host buffers are device-mapped (UVA): x is pulled and y pushed by small kernels
        // chained to the SpMV with programmatic dependent launch, so the SpMV prologue overlaps
        // the x transfer.  Pageable buffers take cudaMemcpyAsync.  (A cached CUDA graph of the
        // memcpy variant measured 11 us slower.)
        auto mapped = [](const void* p) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
                cudaGetLastError();
                return (const void*)nullptr;
            }
            return at.type == cudaMemoryTypeHost ? (const void*)at.devicePointer : (const void*)nullptr;
        };
        const uint16_t* dx = static_cast<const uint16_t*>(mapped(h_x));
        uint16_t* dy = const_cast<uint16_t*>(static_cast<const uint16_t*>(mapped(h_y)));
        if (dx) {
            ck(mk::launch_copy_u16(dx, hx_dev, (uint32_t)m->cols, 1, false, st), "x pull");
            g_launches.fetch_add(1);
        } else {
            ck(cudaMemcpyAsync(hx_dev, h_x, m->cols * 2, cudaMemcpyHostToDevice, st), "H2D x");
        }
        // a mapped host y is written by the SpMV itself, row by row as rows finish (no push step)
        const macko_status sp = spmv_launch(m, hx_dev, hy_dev, st, dx ? MACKO_SPMV_PDL : 0u, dy);
        if (sp != MACKO_OK) fail(sp, g_err);
        if (!dy) ck(cudaMemcpyAsync(h_y, hy_dev, m->rows * 2, cudaMemcpyDeviceToHost, st), "D2H y");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

macko_status macko_dev_validate(const macko_dev_matrix* m, void* stream) {
    return guarded([&] {
        if (!m) fail(MACKO_EINVAL, "null handle");
        DeviceGuard g(m->device);
        device_validate(const_cast<macko_dev_matrix*>(m), (cudaStream_t)stream);
    });
}

macko_status macko_release_cached_memory(void) {
    return guarded([&] { block_cache().trim(); });
}

macko_status macko_dev_free(macko_dev_matrix* m) {
    return guarded([&] {
        if (!m) return;
        DeviceGuard g(m->device);
        delete m;
    });
}

macko_status macko_gen_dense(int device, uint16_t* d_out, uint64_t rows, uint64_t cols, uint64_t ld, uint64_t row0,
                             uint32_t thr24, uint64_t seed, int int_mode, void* stream) {
    return guarded([&] {
        if (!d_out) fail(MACKO_EINVAL, "null output");
        if (ld < cols) fail(MACKO_EINVAL, "leading dimension < cols");
        DeviceGuard g(device);
        ck(mk::launch_gen_dense(d_out, rows, cols, ld, row0, thr24, seed, int_mode, sm_count(device), (cudaStream_t)stream),
           "gen_dense");
        g_launches.fetch_add(1);
    });
}

macko_status macko_gen_vector(int device, uint16_t* d_out, uint64_t n, uint64_t seed, int int_mode, void* stream) {
    return guarded([&] {
        if (!d_out) fail(MACKO_EINVAL, "null output");
        DeviceGuard g(device);
        ck(mk::launch_gen_vector(d_out, n, seed, int_mode, (cudaStream_t)stream), "gen_vector");
        g_launches.fetch_add(1);
    });
}


// ---- MCKO container ----------------------------------------------------------------------
macko_status macko_mcko_write(const char* path, uint64_t rows, uint64_t cols, uint32_t b_delta, const uint16_t* values,
                              uint64_t n_values, const uint8_t* deltas, uint64_t n_delta_bytes, const uint32_t* row_ptrs) {
    return guarded([&] {
        if (!row_ptrs) fail(MACKO_EINVAL, "null row_pointers");
        if (!host_little_endian()) fail(MACKO_EIO, "big-endian host");
        check_bits(b_delta);
        check_shape(rows, cols);
        const uint64_t pad_nnz = row_ptrs[rows];
        if (n_values < pad_nnz || n_delta_bytes * 8 < pad_nnz * b_delta) fail(MACKO_EFORMAT, "arrays shorter than pad_nnz");
        if (pad_nnz && (!values || !deltas)) fail(MACKO_EINVAL, "null payload");
        MckoHeader h;
        h.b_delta = b_delta;
        h.rows = rows;
        h.cols = cols;
        h.pad_nnz = pad_nnz;
        File f(path, "wb");
        write_header(f, h);
        f.write(row_ptrs, (rows + 1) * 4);
        const uint64_t db = delta_bytes(pad_nnz, b_delta), vb = values_bytes(pad_nnz);
        const uint64_t dn = std::min<uint64_t>(n_delta_bytes, db), vn = std::min<uint64_t>(n_values * 2, vb);
        f.write(deltas, dn);
        f.zeros(db - dn);
        f.write(values, vn);
        f.zeros(vb - vn);
    });
}

macko_status macko_mcko_read_info(const char* path, macko_dev_info* out) {
    return guarded([&] {
        if (!out) fail(MACKO_EINVAL, "null argument");
        File f(path, "rb");
        const MckoHeader h = read_header(f);
        std::memset(out, 0, sizeof *out);
        out->rows = h.rows;
        out->cols = h.cols;
        out->pad_nnz = h.pad_nnz;
        out->b_delta = h.b_delta;
        out->values_bytes = values_bytes(h.pad_nnz);
        out->delta_bytes = delta_bytes(h.pad_nnz, h.b_delta);
        out->row_ptr_bytes = 4 * (h.rows + 1);
        out->traffic_bytes = out->values_bytes + out->delta_bytes + out->row_ptr_bytes + 2 * h.cols + 2 * h.rows;
        out->device = -1;
    });
}

macko_status macko_mcko_read(const char* path, uint16_t* values, uint8_t* deltas, uint32_t* row_ptrs) {
    return guarded([&] {
        if (!host_little_endian()) fail(MACKO_EIO, "big-endian host");
        File f(path, "rb");
        const MckoHeader h = read_header(f);
        const std::vector<uint32_t> rp = read_row_ptrs(f, h);
        const uint64_t db = delta_bytes(h.pad_nnz, h.b_delta), vb = values_bytes(h.pad_nnz);
        std::vector<uint8_t> d(db);
        std::vector<uint16_t> v(vb / 2);
        f.read(d.data(), db, "packed_deltas");
        f.read(v.data(), vb, "values");
        host_validate(h, rp, d.data(), v.data());
        if (row_ptrs) std::memcpy(row_ptrs, rp.data(), rp.size() * 4);
        if (deltas) std::memcpy(deltas, d.data(), db);
        if (values) std::memcpy(values, v.data(), vb);
    });
}

macko_status macko_mcko_write_dev(const macko_dev_matrix* m, const char* path, void* stream) {
    return guarded([&] {
        if (!m) fail(MACKO_EINVAL, "null handle");
        if (!host_little_endian()) fail(MACKO_EIO, "big-endian host");
        DeviceGuard g(m->device);
        cudaStream_t st = (cudaStream_t)stream;
        MckoHeader h;
        h.b_delta = m->b_delta;
        h.rows = m->rows;
        h.cols = m->cols;
        h.pad_nnz = m->pad_nnz;
        std::vector<uint32_t> rp(m->rows + 1);
        ck(cudaMemcpyAsync(rp.data(), m->row_ptrs.p, (m->rows + 1) * 4, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        File f(path, "wb");
        write_header(f, h);
        f.write(rp.data(), (m->rows + 1) * 4);
        constexpr size_t kBlock = 32u << 20;
        uint8_t* pinned = nullptr;
        ck(cudaMallocHost(&pinned, kBlock), "pinned staging buffer");
        std::unique_ptr<uint8_t, cudaError_t (*)(void*)> hold(pinned, cudaFreeHost);
        auto dump = [&](const void* src, uint64_t bytes) {
            for (uint64_t off = 0; off < bytes; off += kBlock) {
                const size_t n = (size_t)std::min<uint64_t>(bytes - off, kBlock);
                ck(cudaMemcpyAsync(pinned, static_cast<const uint8_t*>(src) + off, n, cudaMemcpyDeviceToHost, st), "D2H");
                ck(cudaStreamSynchronize(st), "sync");
                f.write(pinned, n);
            }
        };
        dump(m->deltas.p, delta_bytes(m->pad_nnz, m->b_delta));
        dump(m->values.p, values_bytes(m->pad_nnz));
    });
}

macko_status macko_mcko_read_dev(int device, const char* path, void* stream, macko_dev_matrix** out) {
    return guarded([&] {
        if (!out) fail(MACKO_EINVAL, "null argument");
        *out = nullptr;
        if (!host_little_endian()) fail(MACKO_EIO, "big-endian host");
        File f(path, "rb");
        const MckoHeader h = read_header(f);
        std::vector<uint32_t> rp = read_row_ptrs(f, h);
        DeviceGuard g(device);
        cudaStream_t st = (cudaStream_t)stream;
        auto* m = new macko_dev_matrix;
        std::unique_ptr<macko_dev_matrix> hold(m);
        m->device = device;
        m->sms = sm_count(device);
        m->rows = h.rows;
        m->cols = h.cols;
        m->pad_nnz = h.pad_nnz;
        m->b_delta = h.b_delta;
        const uint64_t vb = values_bytes(h.pad_nnz), db = delta_bytes(h.pad_nnz, h.b_delta);
        m->values.alloc(vb / 2 + mk::kChunk);
        m->deltas.alloc(db + mk::kChunk);  // one chunk of codewords at up to 8 bits
        m->row_ptrs.alloc(h.rows + 1);
        ck(cudaMemsetAsync(m->values.p + vb / 2, 0, mk::kChunk * 2, st), "memset");
        ck(cudaMemsetAsync(m->deltas.p + db, 0, mk::kChunk, st), "memset");
        ck(cudaMemcpyAsync(m->row_ptrs.p, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice, st), "upload row_ptrs");
        stream_to_device(f, m->deltas.p, db, st, "packed_deltas");
        stream_to_device(f, m->values.p, vb, st, "values");
        ck(cudaStreamSynchronize(st), "sync");
        m->h_row_ptrs = std::move(rp);
        device_validate(m, st);
        build_plan(m, st);
        *out = hold.release();
    });
}

// ---- Matrix Market ------------------------------------------------------------------------
macko_status macko_mm_read_dense(const char* path, uint64_t* rows, uint64_t* cols, uint16_t* dense) {
    return guarded([&] {
        if (!rows || !cols) fail(MACKO_EINVAL, "null argument");
        read_mm(path, rows, cols, dense);
    });
}


macko_status macko_shard_rows(uint64_t rows, uint32_t n_shards, uint32_t shard, uint64_t* r0, uint64_t* r1) {
    return guarded([&] {
        if (!r0 || !r1 || n_shards == 0 || shard >= n_shards) fail(MACKO_EINVAL, "bad shard request");
        *r0 = rows * shard / n_shards;
        *r1 = rows * (shard + 1) / n_shards;
    });
}

namespace {
// NCCL resolved at run time (no link-time dependency; in a torch process the NCCL it already
// loaded is reused).  nccl.h: ncclResult_t / ncclDataType_t are int enums, ncclComm_t a pointer.
struct NcclApi {
    int (*bcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*allgather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*user_rank)(void*, int*) = nullptr;
    int (*count)(void*, int*) = nullptr;
    const char* (*errstr)(int) = nullptr;
};
constexpr int kNcclFloat16 = 6;  // nccl.h ncclFloat16

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.bcast = reinterpret_cast<decltype(a.bcast)>(dlsym(h, "ncclBroadcast"));
        a.allgather = reinterpret_cast<decltype(a.allgather)>(dlsym(h, "ncclAllGather"));
        a.user_rank = reinterpret_cast<decltype(a.user_rank)>(dlsym(h, "ncclCommUserRank"));
        a.count = reinterpret_cast<decltype(a.count)>(dlsym(h, "ncclCommCount"));
        a.errstr = reinterpret_cast<decltype(a.errstr)>(dlsym(h, "ncclGetErrorString"));
        return a;
    }();
    return api;
}

void nck(int r, const char* what) {
    if (r != 0) fail(MACKO_ENCCL, std::string(what) + ": " + (nccl().errstr ? nccl().errstr(r) : "NCCL error"));
}
}  // namespace

macko_status macko_dev_set_peers(macko_dev_matrix* m, uint16_t* const* peer_y, uint32_t* const* peer_flags, uint32_t n,
                                 void* stream) {
    return guarded([&] {
        if (!m || (n && (!peer_y || !peer_flags))) fail(MACKO_EINVAL, "null argument");
        if (n > mk::kMaxPeers) fail(MACKO_EINVAL, "at most 8 peers");
        DeviceGuard g(m->device);
        mk::PeerTable t{};
        for (uint32_t p = 0; p < n; ++p) {
            if (!peer_y[p] || !peer_flags[p]) fail(MACKO_EINVAL, "null peer pointer");
            t.y[0][p] = t.y[1][p] = peer_y[p];
            t.flag[p] = peer_flags[p];
        }
        (void)stream;  // the table travels in the launch parameters
        m->h_peers = t;
        m->n_peer = n;
    });
}

macko_status macko_dev_set_peer_bank(macko_dev_matrix* m, uint32_t bank, uint16_t* const* peer_y, uint32_t n,
                                     void* stream) {
    return guarded([&] {
        if (!m || !peer_y) fail(MACKO_EINVAL, "null argument");
        if (bank > 1) fail(MACKO_EINVAL, "peer bank must be 0 or 1");
        if (n != m->n_peer || n == 0) fail(MACKO_EINVAL, "set the peers (macko_dev_set_peers) first, same count");
        DeviceGuard g(m->device);
        mk::PeerTable t = m->h_peers;
        for (uint32_t p = 0; p < n; ++p) {
            if (!peer_y[p]) fail(MACKO_EINVAL, "null peer pointer");
            t.y[bank][p] = peer_y[p];
        }
        (void)stream;
        m->h_peers = t;
    });
}

macko_status macko_wait_flags(const uint32_t* d_flags, uint32_t n, uint32_t target, void* stream) {
    return guarded([&] {
        if (!d_flags || n == 0 || n > 32) fail(MACKO_EINVAL, "flags: 1..32 counters");
        ck(mk::launch_wait_flags(d_flags, n, target, (cudaStream_t)stream), "wait_flags");
        g_launches.fetch_add(1);
    });
}

macko_status macko_ipc_get_handle(const void* d_ptr, uint8_t* handle64, uint64_t* offset) {
    return guarded([&] {
        if (!d_ptr || !handle64 || !offset) fail(MACKO_EINVAL, "null argument");
        // the handle names the whole allocation (a caching allocator hands out sub-blocks): the
        // peer opens the base and adds the offset (driver cuMemGetAddressRange, via the runtime's
        // entry-point query, so the library keeps no link-time libcuda dependency)
        using RangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
        static RangeFn range = [] {
            void* f = nullptr;
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                f = nullptr;
            return reinterpret_cast<RangeFn>(f);
        }();
        if (!range) fail(MACKO_ECUDA, "cuMemGetAddressRange unavailable");
        unsigned long long base = 0;
        size_t size = 0;
        if (range(&base, &size, (unsigned long long)reinterpret_cast<uintptr_t>(d_ptr)) != 0)
            fail(MACKO_EINVAL, "not a device allocation");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(handle64, &h, 64);
        *offset = (uint64_t)(reinterpret_cast<uintptr_t>(d_ptr) - base);
    });
}

macko_status macko_ipc_open(const uint8_t* handle64, int device, void** d_ptr) {
    return guarded([&] {
        if (!handle64 || !d_ptr) fail(MACKO_EINVAL, "null argument");
        DeviceGuard g(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, 64);
        ck(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

macko_status macko_ipc_close(void* d_ptr) {
    return guarded([&] {
        if (!d_ptr) fail(MACKO_EINVAL, "null argument");
        ck(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle");
    });
}

macko_status macko_sharded_spmv(const macko_dev_matrix* slab, void* nccl_comm, int root, uint16_t* d_x,
                                uint16_t* d_y, uint64_t rows_total, void* stream) {
    return guarded([&] {
        if (!slab || !nccl_comm || !d_x || !d_y) fail(MACKO_EINVAL, "null argument");
        const NcclApi& api = nccl();
        if (!api.bcast || !api.allgather || !api.user_rank || !api.count)
            fail(MACKO_ENCCL, "libnccl.so.2 not found (macko_sharded_spmv needs NCCL)");
        int n = 0, r = 0;
        nck(api.count(nccl_comm, &n), "ncclCommCount");
        nck(api.user_rank(nccl_comm, &r), "ncclCommUserRank");
        if (n < 1 || rows_total % (uint64_t)n != 0)
            fail(MACKO_EINVAL, "rows_total must split into equal slabs (all-gather of equal counts)");
        const uint64_t slab_rows = rows_total / (uint64_t)n, r0 = slab_rows * (uint64_t)r;
        if (slab->rows != slab_rows) fail(MACKO_EINVAL, "slab rows do not match rows_total / ranks");
        if (root < 0 || root >= n) fail(MACKO_EINVAL, "root out of range");
        DeviceGuard g(slab->device);
        cudaStream_t st = (cudaStream_t)stream;
        nck(api.bcast(d_x, d_x, slab->cols, kNcclFloat16, root, nccl_comm, st), "ncclBroadcast x");
        const macko_status sp = macko_dev_spmv(slab, d_x, d_y + r0, stream);
        if (sp != MACKO_OK) fail(sp, g_err);
        nck(api.allgather(d_y + r0, d_y, slab_rows, kNcclFloat16, nccl_comm, st), "ncclAllGather y");
    });
}

macko_status macko_dev_configure(macko_dev_matrix* m, int x_mode, int ctas_per_sm, void* stream) {
    return guarded([&] {
        if (!m) fail(MACKO_EINVAL, "null handle");
        if (x_mode != -1 && !mk::spmv_valid_config(x_mode, (int)m->b_delta))
            fail(MACKO_EINVAL, "x_mode must be -1 (auto), 0, 1, 6, 7, 8 or 10");
        if (x_mode > 0 && m->cols * 2 > 220 * 1024) fail(MACKO_EINVAL, "x table does not fit shared memory");
        DeviceGuard g(m->device);
        std::lock_guard<std::mutex> lk(m->mu);
        m->force_x_mode = x_mode;
        m->force_ctas = ctas_per_sm;
        build_plan(m, (cudaStream_t)stream);
    });
}

macko_status macko_dev_set_chain_skew(macko_dev_matrix* m, uint32_t start_spread_ns, void* stream) {
    return guarded([&] {
        if (!m) fail(MACKO_EINVAL, "null handle");
        DeviceGuard g(m->device);
        std::lock_guard<std::mutex> lk(m->mu);
        // CTA c of a PDL-chained launch starts ~spread * c / (G-1) after CTA 0; its share is cut by
        // r (1 - 2c/(G-1)) with r = spread / (2 T), T the mean CTA time at ~14 stored elements per
        // ns per CTA (36864x12288 @50 %: 226 M elements, 148 CTAs, ~105 us of walk).
        double r = 0.0;
        if (start_spread_ns && m->pad_nnz && m->grid > 1) {
            const double t_cta_ns = (double)m->pad_nnz / (double)m->grid / 14.0;
            r = std::min(0.45, (double)start_spread_ns / (2.0 * t_cta_ns));
        }
        m->plan_skew = (uint32_t)std::lround(r * 65536.0);
        build_plan(m, (cudaStream_t)stream);
    });
}

macko_status macko_dev_plan_records(const macko_dev_matrix* m, void* recs, uint64_t recs_bytes, void* splits,
                                    uint64_t splits_bytes, void* stream) {
    return guarded([&] {
        if (!m) fail(MACKO_EINVAL, "null handle");
        const uint64_t rb = (uint64_t)m->n_chunks * sizeof(mk::WarpPlan), sb = (uint64_t)m->n_split * 16;
        if ((recs && recs_bytes < rb) || (splits && splits_bytes < sb)) fail(MACKO_EINVAL, "buffer too small");
        DeviceGuard g(m->device);
        cudaStream_t st = (cudaStream_t)stream;
        if (recs && rb) ck(cudaMemcpyAsync(recs, m->plan_recs.p, rb, cudaMemcpyDeviceToHost, st), "D2H");
        if (splits && sb) ck(cudaMemcpyAsync(splits, m->plan_u32.p, sb, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

macko_status macko_dev_launch_info(const macko_dev_matrix* m, macko_launch_info* out) {
    return guarded([&] {
        if (!m || !out) fail(MACKO_EINVAL, "null argument");
        out->grid = (uint32_t)m->grid;
        out->block = mk::kSpmvWarpsPerCta * mk::kWarp;
        out->warps = m->n_chunks;
        out->ctas_per_sm = (uint32_t)m->ctas_per_sm;
        out->n_split_rows = m->n_split;
        out->x_in_smem = (uint32_t)m->x_mode;
        out->n_units = m->n_units;
        out->smem_bytes = m->smem;
        out->reserved0 = 0;
        out->reserved = 0;
    });
}

#ifdef MACKO_TRACE
// trace build only (not declared in include/macko_cuda.h): per-warp prologue timestamps
int macko_trace_read(unsigned long long* host, size_t n) { return (int)mk::trace_read(host, n); }
unsigned macko_trace_slot_counter(void) { return g_trace_slot.load(); }
#endif

}  // extern "C"
