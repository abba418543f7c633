// riann_b200.cu -- C ABI (include/riann_b200.h) over the sm_100a kernels.
//
// Host side of the drop-in boundary: owns device memory for one GPU, keeps the
// reference model and the per-position field resident across frames, and
// launches K1 (units) -> K2 (query) -> pairwise reduction per frame on the
// context's stream.  No CPU fallback: every compute entry point runs on the
// GPU or returns an error.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cub/device/device_segmented_radix_sort.cuh>  // K3 table build only (preprocessing)

#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <array>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "riann_b200.h"
#include "riann_bulk.cuh"
#include "riann_exact_tc.cuh"
#include "riann_effects.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            if (e_ == cudaErrorMemoryAllocation) {                                             \
                cudaGetLastError();                                                            \
                return fail(RIANN_E_CAPACITY, "%s: %s", #call, cudaGetErrorString(e_));        \
            }                                                                                  \
            return fail(RIANN_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                             \
        }                                                                                      \
    } while (0)

#define RET(x)                 \
    do {                       \
        int r_ = (x);          \
        if (r_) return r_;     \
    } while (0)

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes)
    {
        if (bytes <= cap) return 0;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t b = bytes < 256 ? 256 : bytes;
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(RIANN_E_CAPACITY, "cudaMalloc(%zu bytes): %s", b, cudaGetErrorString(e));
        }
        cap = b;
        return 0;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T *as() const
    {
        return static_cast<T *>(p);
    }
};

// numpy pairwise tree over Q values (host-built once per Q).
struct PwTree {
    int64_t q = -1;
    int nleaves = 0, nlevels = 0, nnodes = 0;
    DevBuf leaf_start, leaf_len, leaf_node, level_off, inner, left, right, node_val;

    int build(int64_t Q)
    {
        if (Q == q) return 0;
        std::vector<int64_t> ls;
        std::vector<int32_t> ll, ln, L, R, depth;
        std::vector<std::vector<int32_t>> levels;
        // iterative DFS: node ids assigned in creation order, root 0
        struct Item {
            int64_t s, n;
            int id, dep;
        };
        std::vector<Item> st;
        L.push_back(-1);
        R.push_back(-1);
        st.push_back({0, Q, 0, 0});
        int nid = 1;
        while (!st.empty()) {
            Item it = st.back();
            st.pop_back();
            if (it.n <= 128) {
                ls.push_back(it.s);
                ll.push_back((int32_t)it.n);
                ln.push_back(it.id);
            } else {
                int64_t h = it.n / 2;
                h -= h % 8;
                int a = nid++, b = nid++;
                L.push_back(-1);
                R.push_back(-1);
                L.push_back(-1);
                R.push_back(-1);
                L[it.id] = a;
                R[it.id] = b;
                if ((int)levels.size() <= it.dep) levels.resize(it.dep + 1);
                levels[it.dep].push_back(it.id);
                st.push_back({it.s, h, a, it.dep + 1});
                st.push_back({it.s + h, it.n - h, b, it.dep + 1});
            }
        }
        std::vector<int32_t> off(1, 0), inner_ids;
        for (int d = (int)levels.size() - 1; d >= 0; d--) {
            for (int x : levels[d]) inner_ids.push_back(x);
            off.push_back((int32_t)inner_ids.size());
        }
        nleaves = (int)ls.size();
        nlevels = (int)levels.size();
        nnodes = nid;
        RET(leaf_start.ensure(ls.size() * 8));
        RET(leaf_len.ensure(ll.size() * 4));
        RET(leaf_node.ensure(ln.size() * 4));
        RET(level_off.ensure(off.size() * 4));
        RET(inner.ensure((inner_ids.size() + 1) * 4));
        RET(left.ensure(L.size() * 4));
        RET(right.ensure(R.size() * 4));
        RET(node_val.ensure((size_t)nid * 8));
        CK(cudaMemcpy(leaf_start.p, ls.data(), ls.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(leaf_len.p, ll.data(), ll.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(leaf_node.p, ln.data(), ln.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(level_off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
        if (!inner_ids.empty())
            CK(cudaMemcpy(inner.p, inner_ids.data(), inner_ids.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(left.p, L.data(), L.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(right.p, R.data(), R.size() * 4, cudaMemcpyHostToDevice));
        q = Q;
        return 0;
    }
};

// frame phases timed by riann_timing_phases (RIANN_NPHASES in the header)
enum { PH_UNITS, PH_P0A, PH_P0B, PH_DRAW, PH_GROUP, PH_WINDOW, PH_FILTER, PH_FINAL, PH_TAIL, PH_QUERY };
const char *const kPhaseNames[RIANN_NPHASES] = {"riann:units", "riann:p0a", "riann:p0b", "riann:draw",
                                                "riann:group", "riann:window", "riann:filter", "riann:final",
                                                "riann:tail", "riann:query"};

// Per-stream device state: the previous field and the previous frame's unit
// rows (double-buffered) plus the replay snapshot.  A context holds one active
// slot and parks the others, so interleaved streams on one GPU (bands of one
// frame, two clips) never read each other's field or units.
struct StreamState {
    DevBuf units[2], fld_idx[2], fld_dist, snap_idx, snap_units;
    int cur_units = 0, cur_fld = 0;
    bool have_prev_units = false;
    int64_t prev_units_rows = 0, field_count = -1;
    int64_t snap_field = -1, snap_units_rows = 0;
    bool snap_have_units = false, snap_valid = false;
    void release()
    {
        for (DevBuf *b : {&units[0], &units[1], &fld_idx[0], &fld_idx[1], &fld_dist, &snap_idx, &snap_units})
            b->release();
        *this = StreamState();
    }
};

}  // namespace

struct riann_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;  // heavy-query fallback, concurrent with the ring phases
    cudaStream_t stream3 = nullptr;  // final-scan projection, concurrent with P0 / ring phases
    cudaEvent_t ev_p0 = nullptr, ev_heavy = nullptr, ev_units = nullptr, ev_proj = nullptr, ev_tc = nullptr;
    int sms = 0;
    int smem_optin = 0;
    // model
    int64_t n = 0;
    int dim = 0, pw = 0, ph = 0, C = 1;
    bool tables = false;
    bool idx16 = false;  // sorted index table stored as uint16 (n <= 65536)
    DevBuf refs, refs16, err16, sdist, sidx, dmat;
    DevBuf pos, coarse, coarse1;  // rank rows and two-level coarse index (bulk path, n <= 65536)
    // row-sharded tables (riann_model_attach_shards): device arrays of the
    // shards' sdist / sidx / dmat base pointers; own_row0/own_rows: the rows
    // this context's own tables hold
    int nshards = 0;
    int64_t shard_rows = 0, own_row0 = 0, own_rows = -1;
    DevBuf sh_ptrs;
    // PCA screening basis (bulk final scan)
    DevBuf pca_T, refs_pca16, e16p, units_pca, e16max;
    bool pca = false;
    float pca_dq = 0.f, pca_eta = 0.f, pca_e16max = 0.f;
    int ncoarse = 0, cs1 = 0;
    bool bulk_disabled = false;
    // K4 tensor-core comparator: split reference operand, norms, per-call scratch
    bool exact_simt = false, x_ready = false;
    DevBuf fx_frame, fx_idx, fx_pay, fx_norm, fx_out, fx_rgb, pack;
    DevBuf x_B, x_nr, x_center, x_scal, x_A, x_nq, x_cand, x_lb, x_ncand, x_ub, x_fb, x_q, x_idx, x_dist;
    uint64_t x_checked = 0, x_fallback = 0;
    // bulk-path frame buffers
    DevBuf b_state, b_pool, b_bits, b_kept, b_active[2], b_heavy, b_heavy2, b_heavy3, b_counters, b_counts, b_starts,
        b_gdesc, overflow2;
    // frame path
    DevBuf frame, units[2], prev, fld_idx[2], fld_dist, tc, tc_sum, stats, err, overflow, keys, kw, koff;
    DevBuf q_rings, q_evals, q_cand, q_first, q_scanned, q_scanned_len, small;
    int cur_units = 0;
    bool have_prev_units = false;
    int64_t prev_units_rows = 0;
    int cur_fld = 0;
    int64_t field_count = -1;
    // stream slots (riann_slot_select): the active slot's state lives in the
    // members above and below, the others are parked here
    int slot = 0;
    std::map<int, StreamState> parked;
    PwTree tree;
    // state snapshot (riann_state_save / riann_state_restore)
    DevBuf snap_idx, snap_units;
    int64_t snap_field = -1, snap_units_rows = 0;
    bool snap_have_units = false, snap_valid = false;
    // per-kernel event timing of the frame path (riann_timing_*)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::array<cudaEvent_t, 4>> ev_pending;
    double t_ms[3] = {0, 0, 0};
    uint64_t t_frames = 0, launches = 0;
    // per-phase event marks of the frame in flight (label, event) and of the
    // frames not yet read; summed per label by riann_timing_read
    std::vector<std::pair<int, cudaEvent_t>> marks;
    std::vector<std::vector<std::pair<int, cudaEvent_t>>> marks_pending;
    double t_phase[RIANN_NPHASES] = {};
    std::vector<std::array<double, RIANN_NPHASES>> t_phase_frames;  // per timed frame
    bool nvtx_open = false;

    cudaEvent_t ev()
    {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }

    int use()
    {
        CK(cudaSetDevice(device));
        return 0;
    }
    // exchange the active stream state with `o`
    void swap_state(StreamState &o)
    {
        for (int k = 0; k < 2; k++) {
            std::swap(units[k], o.units[k]);
            std::swap(fld_idx[k], o.fld_idx[k]);
        }
        std::swap(fld_dist, o.fld_dist);
        std::swap(snap_idx, o.snap_idx);
        std::swap(snap_units, o.snap_units);
        std::swap(cur_units, o.cur_units);
        std::swap(cur_fld, o.cur_fld);
        std::swap(have_prev_units, o.have_prev_units);
        std::swap(prev_units_rows, o.prev_units_rows);
        std::swap(field_count, o.field_count);
        std::swap(snap_field, o.snap_field);
        std::swap(snap_units_rows, o.snap_units_rows);
        std::swap(snap_have_units, o.snap_have_units);
        std::swap(snap_valid, o.snap_valid);
    }
    uint64_t bytes() const
    {
        uint64_t b = refs.cap + refs16.cap + err16.cap + dmat.cap + pos.cap + coarse.cap + coarse1.cap + b_state.cap + pca_T.cap +
                     refs_pca16.cap + e16p.cap + units_pca.cap +
                     b_pool.cap + sdist.cap + sidx.cap + frame.cap + units[0].cap + units[1].cap + prev.cap +
                     fld_idx[0].cap + fld_idx[1].cap + fld_dist.cap + tc.cap + overflow.cap + keys.cap + x_B.cap + x_A.cap +
                     x_cand.cap + x_lb.cap + snap_idx.cap + snap_units.cap;
        for (const auto &kv : parked) {
            const StreamState &st = kv.second;
            b += st.units[0].cap + st.units[1].cap + st.fld_idx[0].cap + st.fld_idx[1].cap + st.fld_dist.cap +
                 st.snap_idx.cap + st.snap_units.cap;
        }
        return b;
    }
};

namespace {

// Mark the start of a frame phase on the ctx stream: a CUDA event while
// timing is on (riann_timing_phases) and an NVTX range (ncu --nvtx / nsys).
// label < 0 closes the last phase.
void tmark(riann_ctx *c, int label)
{
    if (c->nvtx_open) {
        nvtxRangePop();
        c->nvtx_open = false;
    }
    if (label >= 0) {
        nvtxRangePushA(kPhaseNames[label]);
        c->nvtx_open = true;
    }
    if (!c->timing) return;
    cudaEvent_t e = c->ev();
    cudaEventRecord(e, c->stream);
    c->marks.push_back({label, e});
}

template <int D, class IdxT>
int launch_query_t(riann_ctx *c, rb::QueryParams &P)
{
    const size_t per_warp = (size_t)rb::K2_SMEM_BYTES;
    const int wpb = 8;
    const size_t smem = per_warp * wpb;
    using LT = typename std::conditional<sizeof(IdxT) == 2, uint16_t, uint32_t>::type;
    auto kern = rb::query_kernel<D, IdxT, LT>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, wpb * 32, smem));
    if (bps < 1) bps = 1;
    int64_t blocks = (int64_t)c->sms * bps;
    int64_t need = (P.Q + wpb - 1) / wpb;
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    RET(c->overflow.ensure((size_t)blocks * wpb * 2 * (size_t)c->n * (c->idx16 ? 2 : 4)));
    P.overflow = c->overflow.as<uint32_t>();
    kern<<<(unsigned)blocks, wpb * 32, smem, c->stream>>>(P);
    CK(cudaGetLastError());
    return 0;
}

template <class IdxT>
int launch_query_i(riann_ctx *c, rb::QueryParams &P)
{
    switch (c->dim) {
    case 16: return launch_query_t<16, IdxT>(c, P);
    case 64: return launch_query_t<64, IdxT>(c, P);
    case 192: return launch_query_t<192, IdxT>(c, P);
    default: return launch_query_t<0, IdxT>(c, P);
    }
}

// P0-heavy queries the per-query kernel takes on the second stream; more than
// this (a stream's first frame) run further bulk passes instead
constexpr int64_t K2CAP = 16384;

template <int D>
int run_bulk_t(riann_ctx *c, rb::QueryParams &Pq)
{
    const int64_t QN = Pq.Q, n = c->n;
    RET(c->b_state.ensure((size_t)QN * sizeof(rb::QState)));
    // candidate pool: sum of first-ring sizes, capped (overflowing queries fall back to K2)
    // candidate pool (u16 entries + two alive-bit buffers, 2.25 B per entry): up
    // to 8,192 entries per query and 16 G entries, within 40 % of the free HBM
    // (with what the pool already holds); a first frame whose first rings do
    // not fit takes further passes
    size_t pool_entries = std::min<size_t>((size_t)QN * 8192, (size_t)16 << 30);
    if (pool_entries * 2 > c->b_pool.cap) {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const size_t budget = (size_t)((double)(fr + c->b_pool.cap + c->b_bits.cap) * 0.4 / 2.25);
        pool_entries = std::max<size_t>(std::min(pool_entries, budget), std::min<size_t>(pool_entries, (size_t)1 << 24));
        pool_entries = std::max<size_t>(pool_entries, c->b_pool.cap / 2);
    } else {
        pool_entries = c->b_pool.cap / 2;
    }
    pool_entries &= ~(size_t)127;
    RET(c->b_pool.ensure(pool_entries * 2));
    RET(c->b_bits.ensure(pool_entries / 4));  // two alive-bit buffers
    RET(c->b_kept.ensure((size_t)QN * 4));
    RET(c->b_active[0].ensure((size_t)QN * 4));
    RET(c->b_active[1].ensure((size_t)QN * 4));
    RET(c->b_heavy.ensure((size_t)QN * 4));
    RET(c->b_heavy2.ensure((size_t)QN * 4));
    RET(c->b_gdesc.ensure((size_t)QN * 16));
    RET(c->b_counters.ensure(256));
    RET(c->b_counts.ensure((size_t)(n + 1) * 4));
    RET(c->b_starts.ensure((size_t)(n + 1) * 4));
    // [0..1] active counts, [2] P0 heavy, [3] item counter, [4..5] pool top, [6] ring heavy,
    // [7] P0 heavy count handed to the second stream
    int32_t *ctr = c->b_counters.as<int32_t>();
    CK(cudaMemsetAsync(ctr, 0, 256, c->stream));

    rb::BulkParams B;
    memset(&B, 0, sizeof B);
    B.refs = c->refs.as<float>();
    B.refs16 = c->refs16.as<__half>();
    B.err16 = c->err16.as<float>();
    B.sdist = c->sdist.as<float>();
    B.sidx = c->sidx.as<uint16_t>();
    B.pos = c->pos.as<uint16_t>();
    B.coarse = c->coarse.as<float>();
    B.coarse1 = c->coarse1.as<float>();
    B.cs1 = c->cs1;
    B.vec_probe = (c->cs1 % 4 == 0 && c->ncoarse % 4 == 0 && n % 64 == 0) ? 1 : 0;
    B.n = n;
    B.ncoarse = c->ncoarse;
    B.units = Pq.units;
    B.prev = Pq.prev;
    B.Q = QN;
    B.seed_lo = Pq.seed_lo;
    B.seed_hi = Pq.seed_hi;
    B.seed_nw = Pq.seed_nw;
    B.gw = Pq.gw;
    B.gy0 = Pq.gy0;
    B.t = Pq.t;
    B.L = Pq.L;
    B.alpha = Pq.alpha;
    B.max_rings = Pq.max_rings;
    B.passes = Pq.passes;
    B.st = c->b_state.as<rb::QState>();
    B.pool = c->b_pool.as<uint16_t>();
    B.pool_top = reinterpret_cast<unsigned long long *>(ctr + 4);
    B.pool_cap = (int64_t)pool_entries;
    B.bits0 = c->b_bits.as<uint8_t>();
    B.bits1 = B.bits0 + pool_entries / 8;
    B.kept = c->b_kept.as<int32_t>();
    B.heavy = c->b_heavy.as<int32_t>();
    B.n_heavy = ctr + 2;
    B.counts = c->b_counts.as<int32_t>();
    B.starts = c->b_starts.as<int32_t>();
    B.gdesc = c->b_gdesc.as<int4>();
    B.item_next = ctr + 3;
    B.fdirect = QN < 8 * n ? rb::FDIRECT : 0;  // few queries per anchor (a row band)
    B.out_idx = Pq.out_idx;
    B.out_dist = Pq.out_dist;
    B.stats = Pq.stats;
    B.err = Pq.err;

    // projection for the final scan (q' = T^T q, fp32 SIMT GEMM) on a third
    // stream: it needs only the unit rows, so it overlaps P0 and the rings
    RET(c->units_pca.ensure((size_t)QN * D * 4));
    CK(cudaEventRecord(c->ev_units, c->stream));
    CK(cudaStreamWaitEvent(c->stream3, c->ev_units, 0));
    {
        using CF = rb::ProjCfg<D>;
        const int64_t tiles = (QN + CF::PQ - 1) / CF::PQ;
        int bps = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, rb::proj_kernel<D>, CF::THREADS, 0));
#ifndef RIANN_PROJ_PERSIST
#define RIANN_PROJ_PERSIST 0
#endif
        // one tile per CTA (not persistent): with the side stream at low priority the
        // block scheduler gives freed SM slots to the frame kernels first
        const int64_t grid = RIANN_PROJ_PERSIST ? std::min<int64_t>(tiles, (int64_t)c->sms * std::max(bps, 1)) : tiles;
        rb::proj_kernel<D><<<(unsigned)std::max<int64_t>(grid, 1), CF::THREADS, 0, c->stream3>>>(
            Pq.units, c->pca_T.as<float>(), QN, c->units_pca.as<float>());
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->ev_proj, c->stream3));
        c->launches += 1;
    }
    auto dk = rb::bulk_draw_kernel<D>;
    int d_bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d_bps, dk, 256, 0));
    const unsigned d_grid = (unsigned)(c->sms * std::max(d_bps, 1));
    auto fk = rb::bulk_filter_kernel;
    const size_t fsmem = rb::filter_smem(n);
    CK(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
    int f_bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f_bps, fk, rb::FW2 * 32, fsmem));
    const unsigned f_grid = (unsigned)(c->sms * std::max(f_bps, 1));
    const unsigned small_grid = (unsigned)c->sms * 4;
    auto wk = rb::bulk_window_kernel<D>;
    int w_bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&w_bps, wk, 256, 0));
    const unsigned w_grid = (unsigned)(c->sms * std::max(w_bps, 1));
    int32_t *ring_heavy = c->b_heavy2.as<int32_t>();  // > BULK_U used anchors: K2 from scratch, all passes

    // One pass of the bulk path over the queries qin[0 .. nin) (all queries when
    // qin is null): P0a allocates lists from an empty pool; queries that do not
    // fit go to heavy_out (count at ctr[2]).
    auto one_pass = [&](const int32_t *qin, int64_t nin, int32_t *heavy_out, bool first_pass) -> int {
        B.qin = qin;
        B.n_qin = nin;
        B.heavy = heavy_out;
        B.n_heavy = ctr + 2;
        if (!first_pass) {
            CK(cudaMemsetAsync(ctr, 0, 4 * 4, c->stream));   // active counts, heavy count, item counter
            CK(cudaMemsetAsync(ctr + 4, 0, 8, c->stream));   // pool top
        }
        // P0a: d_prev, first-ring windows, list allocation (four queries per warp)
        tmark(c, PH_P0A);
        {
            auto k = rb::bulk_p0a_kernel<D>;
            int bps = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, 256, 0));
            k<<<(unsigned)(c->sms * std::max(bps, 1)), 256, 0, c->stream>>>(B);
            CK(cudaGetLastError());
            c->launches += 1;
        }
        if (first_pass) {
            // the first K2CAP queries P0 could not take (first ring > LIGHT_MAX, pool
            // full) run the per-query kernel on the second stream while the ring
            // phases proceed; more than that (the first frame of a stream: random
            // prev, first rings of ~70 % of n) take further bulk passes
            // its count is copied (ctr[7]): later passes reuse ctr[2]
            CK(cudaMemcpyAsync(ctr + 7, ctr + 2, 4, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaEventRecord(c->ev_p0, c->stream));
            CK(cudaStreamWaitEvent(c->stream2, c->ev_p0, 0));
            rb::QueryParams H = Pq;
            H.qlist = heavy_out;
            H.n_qlist = ctr + 7;
            H.qlist_cap = K2CAP;
            cudaStream_t main = c->stream;
            c->stream = c->stream2;
            DevBuf keep = c->overflow;
            c->overflow = c->overflow2;
            const int r = c->idx16 ? launch_query_i<uint16_t>(c, H) : launch_query_i<int32_t>(c, H);
            c->overflow2 = c->overflow;
            c->overflow = keep;
            c->stream = main;
            RET(r);
            c->launches += 1;
        }
        // P0b: sorted fixed lists + alive bits (warp per query, bitmap in shared memory)
        tmark(c, PH_P0B);
        {
            const int wpb = RIANN_P0_WPB;
            const size_t smem = (size_t)wpb * rb::p0_smem_words(n) * 4;
            auto k = rb::bulk_p0_kernel<D>;
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int bps = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, wpb * 32, smem));
            int64_t blocks = std::min<int64_t>((int64_t)c->sms * std::min(std::max(bps, 1), 8), (QN + wpb - 1) / wpb);
            B.active_out = c->b_active[0].as<int32_t>();
            B.n_active_out = ctr + 0;
            k<<<(unsigned)std::max<int64_t>(blocks, 1), wpb * 32, smem, c->stream>>>(B);
            CK(cudaGetLastError());
            c->launches += 1;
        }
        // first anchors (search.py:119-133): the draw kernel seeds each key's generator
        tmark(c, PH_DRAW);
        B.heavy = ring_heavy;
        B.n_heavy = ctr + 6;
        CK(cudaMemsetAsync(B.counts, 0, (size_t)(n + 1) * 4, c->stream));  // the draw counts anchors
        dk<<<d_grid, 256, 0, c->stream>>>(B, 1);
        CK(cudaGetLastError());
        c->launches += 1;
        if (first_pass) CK(cudaEventRecord(c->ev_heavy, c->stream2));
        // ring phases: group by anchor -> filter (anchor rows through shared memory) -> draw
        const int phases = Pq.max_rings - 1;
        for (int ph = 0; ph < phases; ph++) {
            const int in = ph & 1, out = in ^ 1;
            B.active_in = c->b_active[in].as<int32_t>();
            B.n_active_in = ctr + in;
            B.active_out = c->b_active[out].as<int32_t>();
            B.n_active_out = ctr + out;
            if (ph >= 15) {  // long ring caps: stop once no query is left
                int32_t h = 0;
                CK(cudaMemcpyAsync(&h, ctr + in, 4, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
                if (h == 0) break;
            }
            CK(cudaMemsetAsync(ctr + out, 0, 4, c->stream));
            CK(cudaMemsetAsync(ctr + 3, 0, 4, c->stream));
            tmark(c, PH_GROUP);
#ifndef RIANN_COMPACT
#define RIANN_COMPACT 1
#endif
            // tiny frames are launch-bound: skip; with one phase left the criterion cannot hold
            if (RIANN_COMPACT && ph >= 1 && QN >= 16384 && 2 * (phases - ph) > RIANN_COMPACT_X2) {
                // dense lists (mostly dead by now) are rewritten before the phases left read them again
                rb::bulk_compact_kernel<<<(unsigned)c->sms * 8, 256, 0, c->stream>>>(B, phases - ph);
                CK(cudaGetLastError());
                c->launches += 1;
            }
            rb::anchor_scan_kernel<<<1, rb::SCAN_T, 0, c->stream>>>(B.counts, B.starts, (int)(n + 1));
            CK(cudaGetLastError());
            rb::bulk_scatter_kernel<<<small_grid, 256, 0, c->stream>>>(B);
            CK(cudaGetLastError());
            tmark(c, PH_WINDOW);
            wk<<<w_grid, 256, 0, c->stream>>>(B);
            CK(cudaGetLastError());
            tmark(c, PH_FILTER);
            fk<<<f_grid, rb::FW2 * 32, fsmem, c->stream>>>(B, ph & 1);
            CK(cudaGetLastError());
            tmark(c, PH_DRAW);
            CK(cudaMemsetAsync(B.counts, 0, (size_t)(n + 1) * 4, c->stream));  // the draw counts anchors
            dk<<<d_grid, 256, 0, c->stream>>>(B, ph & 1);
            CK(cudaGetLastError());
            c->launches += 5;
        }
        // final scan of the light queries (PCA-basis screening)
        tmark(c, PH_FINAL);
        {
            CK(cudaStreamWaitEvent(c->stream, c->ev_proj, 0));
            rb::ScreenParams SP;
            SP.refs_pca16 = c->refs_pca16.as<__half>();
            SP.e16p = c->e16p.as<float>();
            SP.units_pca = c->units_pca.as<float>();
            SP.dq = c->pca_dq + 1e-12f;
            SP.slack = c->pca_dq + c->pca_e16max + 2e-12f;
            SP.one_plus_eta = 1.0f + c->pca_eta * 1.001f;
            SP.one_minus_eta = 1.0f - c->pca_eta * 1.001f;
            auto k = rb::bulk_final_kernel<D>;
            const size_t smem = 8 * rb::final_warp_bytes();
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int bps = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, 256, smem));
            int64_t blocks = std::min<int64_t>((int64_t)c->sms * std::max(bps, 1), (QN + 7) / 8);
            k<<<(unsigned)std::max<int64_t>(blocks, 1), 256, smem, c->stream>>>(B, SP);
            CK(cudaGetLastError());
            c->launches += 1;
        }
        return 0;
    };
    RET(one_pass(nullptr, 0, c->b_heavy.as<int32_t>(), true));
    // more P0-heavy queries than K2CAP: bulk passes over the rest, pool reset each time
    {
        int32_t nh = 0;
        CK(cudaMemcpyAsync(&nh, ctr + 2, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (nh > K2CAP) {
            // b_heavy[0 .. K2CAP) stays with the second stream's K2; later passes
            // alternate between the two halves of b_heavy3
            const int64_t rest = nh - K2CAP;
            RET(c->b_heavy3.ensure((size_t)rest * 8));
            int32_t *bufs[2] = {c->b_heavy3.as<int32_t>(), c->b_heavy3.as<int32_t>() + rest};
            const int32_t *qin = c->b_heavy.as<int32_t>() + K2CAP;
            int64_t nin = rest;
            for (int pass = 0; nin > 0; pass++) {
                int32_t *hout = bufs[pass & 1];
                RET(one_pass(qin, nin, hout, false));
                int32_t nout = 0;
                CK(cudaMemcpyAsync(&nout, ctr + 2, 4, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
                if (nout == 0) break;
                if (nout >= nin) {
                    // no progress (first rings > LIGHT_MAX or alone larger than the pool): K2
                    rb::QueryParams H = Pq;
                    H.qlist = hout;
                    H.n_qlist = ctr + 2;
                    const int r = c->idx16 ? launch_query_i<uint16_t>(c, H) : launch_query_i<int32_t>(c, H);
                    RET(r);
                    c->launches += 1;
                    break;
                }
                qin = hout;
                nin = nout;
            }
        }
    }
    // ring-phase stragglers (> BULK_U used anchors in S): per-query kernel from
    // scratch on the main stream, then join the second stream
    Pq.qlist = ring_heavy;
    Pq.n_qlist = ctr + 6;
    tmark(c, PH_TAIL);
    CK(cudaStreamWaitEvent(c->stream, c->ev_heavy, 0));
    return 1;
}

int launch_query(riann_ctx *c, rb::QueryParams &P)
{
    P.refs16 = c->refs16.as<__half>();
    P.err16 = c->err16.as<float>();
    P.dmat = c->dmat.as<float>();
    P.pos = (c->nshards == 0 && c->idx16 && c->pos.p) ? c->pos.as<uint16_t>() : nullptr;
    if (c->nshards > 0) {
        // row-sharded tables: the per-query kernel reads rows through the shard table
        const void *const *sp = c->sh_ptrs.as<const void *const>();
        P.sh_sdist = reinterpret_cast<const float *const *>(sp);
        P.sh_sidx = sp + c->nshards;
        P.sh_dmat = reinterpret_cast<const float *const *>(sp + 2 * c->nshards);
        P.shard_rows = c->shard_rows;
        P.nshards = c->nshards;
        P.sdist = nullptr;
        P.sidx = nullptr;
        P.dmat = nullptr;
    }
    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < c->n) bits++;
    P.passes = (bits + 7) / 8;
    if (!P.qlist && !P.key_words && !P.scanned && c->nshards == 0 && c->idx16 && c->pos.p && c->pca &&
        !c->bulk_disabled &&
        (c->dim == 64 || c->dim == 192) && c->n % 16 == 0) {
        int r = c->dim == 64 ? run_bulk_t<64>(c, P) : run_bulk_t<192>(c, P);
        if (r != 1) return r;
        // falls through: P.qlist = heavy queries
    }
    return c->idx16 ? launch_query_i<uint16_t>(c, P) : launch_query_i<int32_t>(c, P);
}

int check_model(riann_ctx *c, bool need_tables)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (c->n <= 0) return fail(RIANN_E_STATE, "no reference model uploaded");
    if (need_tables && !c->tables) return fail(RIANN_E_STATE, "model has no sorted tables");
    return 0;
}

int check_err(riann_ctx *c)
{
    int h = 0;
    CK(cudaMemcpyAsync(&h, c->err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
#ifdef RIANN_BOUNDS
    {
        CK(cudaDeviceSynchronize());
        unsigned site = 0, zero = 0;
        CK(cudaMemcpyFromSymbol(&site, rb::rb_bounds_site, 4));
        if (site) {
            CK(cudaMemcpyToSymbol(rb::rb_bounds_site, &zero, 4));
            return fail(RIANN_E_CUDA, "device bounds check failed at site %u", site);
        }
    }
#endif
    if (h == rb::ERR_PREV_RANGE) return fail(RIANN_E_INDEX, "prev_index out of range for %lld references", (long long)c->n);
    if (h == rb::ERR_USED_OVERFLOW)
        return fail(RIANN_E_UNSUPPORTED, "more than 128 used anchors remained in the candidate set");
    if (h) return fail(RIANN_E_CUDA, "kernel error %d", h);
    return 0;
}

// Cyclic Jacobi eigendecomposition of a symmetric matrix (row-major, dim D):
// A is destroyed, V receives eigenvectors as columns, w the eigenvalues.
void jacobi_eigen(std::vector<double> &A, int D, std::vector<double> &V, std::vector<double> &w)
{
    V.assign((size_t)D * D, 0.0);
    for (int i = 0; i < D; i++) V[(size_t)i * D + i] = 1.0;
    double total = 0.0;
    for (double x : A) total += x * x;
    for (int sweep = 0; sweep < 60; sweep++) {
        double off = 0.0;
        for (int p = 0; p < D; p++)
            for (int q = p + 1; q < D; q++) off += A[(size_t)p * D + q] * A[(size_t)p * D + q];
        if (off <= 1e-24 * total || off == 0.0) break;
        for (int p = 0; p < D; p++) {
            for (int q = p + 1; q < D; q++) {
                const double apq = A[(size_t)p * D + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double app = A[(size_t)p * D + p], aqq = A[(size_t)q * D + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < D; k++) {
                    const double akp = A[(size_t)k * D + p], akq = A[(size_t)k * D + q];
                    A[(size_t)k * D + p] = cs * akp - sn * akq;
                    A[(size_t)k * D + q] = sn * akp + cs * akq;
                }
                for (int k = 0; k < D; k++) {
                    const double apk = A[(size_t)p * D + k], aqk = A[(size_t)q * D + k];
                    A[(size_t)p * D + k] = cs * apk - sn * aqk;
                    A[(size_t)q * D + k] = sn * apk + cs * aqk;
                }
                for (int k = 0; k < D; k++) {
                    const double vkp = V[(size_t)k * D + p], vkq = V[(size_t)k * D + q];
                    V[(size_t)k * D + p] = cs * vkp - sn * vkq;
                    V[(size_t)k * D + q] = sn * vkp + cs * vkq;
                }
            }
        }
    }
    w.resize(D);
    for (int i = 0; i < D; i++) w[i] = A[(size_t)i * D + i];
}

// PCA screening basis of the references (speed only: any orthogonal basis
// gives exact results; the bounds account for T's non-orthogonality).
int build_pca(riann_ctx *c, const float *refs_host)
{
    c->pca = false;
    const int D = c->dim;
    const int64_t n = c->n;
    if (!(D == 64 || D == 192)) return 0;
    const int64_t step = std::max<int64_t>(1, n / 16384);
    std::vector<double> mu(D, 0.0), C((size_t)D * D, 0.0);
    int64_t m = 0;
    for (int64_t j = 0; j < n; j += step, m++)
        for (int i = 0; i < D; i++) mu[i] += refs_host[j * D + i];
    for (int i = 0; i < D; i++) mu[i] /= (double)m;
    std::vector<double> x(D);
    for (int64_t j = 0; j < n; j += step) {
        for (int i = 0; i < D; i++) x[i] = refs_host[j * D + i] - mu[i];
        for (int a = 0; a < D; a++) {
            const double xa = x[a];
            double *row = &C[(size_t)a * D];
            for (int b = a; b < D; b++) row[b] += xa * x[b];
        }
    }
    for (int a = 0; a < D; a++)
        for (int b = 0; b < a; b++) C[(size_t)a * D + b] = C[(size_t)b * D + a];
    std::vector<double> V, w;
    jacobi_eigen(C, D, V, w);
    std::vector<int> order(D);
    for (int i = 0; i < D; i++) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return w[a] > w[b]; });
    std::vector<float> T((size_t)D * D);  // T[k][i]: entry k of basis vector i
    for (int k = 0; k < D; k++)
        for (int i = 0; i < D; i++) T[(size_t)k * D + i] = (float)V[(size_t)k * D + order[i]];
    // eta >= ||T^T T - I||_2 (Frobenius bound, float64)
    double fro = 0.0;
    for (int a = 0; a < D; a++)
        for (int b = 0; b < D; b++) {
            double dot = 0.0;
            for (int k = 0; k < D; k++) dot += (double)T[(size_t)k * D + a] * (double)T[(size_t)k * D + b];
            const double e = dot - (a == b ? 1.0 : 0.0);
            fro += e * e;
        }
    const double eta = std::sqrt(fro) * 1.01 + 1e-12;
    if (eta > 1e-3) return 0;  // basis too far from orthogonal: skip PCA screening
    // fp32 GEMM error bound for q' = T^T q (proj_kernel, any summation order), ||q|| <= 1 + 1e-6: per component
    // gamma_D * sum_k |T_ki q_k| <= gamma_D * ||T_.i|| * ||q||
    const double u = std::ldexp(1.0, -24), gam = D * u / (1.0 - D * u);
    const double dq = gam * std::sqrt((double)D) * std::sqrt(1.0 + eta) * (1.0 + 1e-6) * 1.01 + 1e-12;
    RET(c->pca_T.ensure((size_t)D * D * 4));
    RET(c->refs_pca16.ensure((size_t)n * D * 2));
    RET(c->e16p.ensure((size_t)n * 4));
    RET(c->e16max.ensure(16));
    CK(cudaMemcpyAsync(c->pca_T.p, T.data(), (size_t)D * D * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->e16max.p, 0, 16, c->stream));
    rb::refs_pca_kernel<<<(unsigned)((n + 127) / 128), 128, 0, c->stream>>>(
        c->refs.as<float>(), c->pca_T.as<float>(), n, D, c->refs_pca16.as<__half>(), c->e16p.as<float>(),
        c->e16max.as<unsigned>());
    CK(cudaGetLastError());
    unsigned mx = 0;
    CK(cudaMemcpyAsync(&mx, c->e16max.p, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float e16m;
    memcpy(&e16m, &mx, 4);
    c->pca_dq = (float)dq;
    c->pca_eta = (float)eta;
    c->pca_e16max = e16m;
    c->pca = true;
    return 0;
}

// rank rows + coarse index for the bulk path (needs the u16 index table)
int build_bulk_tables(riann_ctx *c)
{
    if (!c->idx16) return 0;
    const int64_t n = c->n;
    c->ncoarse = (int)((n + rb::COARSE - 1) / rb::COARSE);
    RET(c->pos.ensure((size_t)n * n * 2));
    RET(c->coarse.ensure((size_t)n * c->ncoarse * 4));
    const int64_t chunk = std::max<int64_t>(1, (int64_t)((1ull << 28) / (size_t)n));
    for (int64_t r0 = 0; r0 < n; r0 += chunk) {
        const int64_t rows = std::min<int64_t>(chunk, n - r0);
        const int64_t m = rows * n;
        rb::pos_scatter_kernel<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(
            c->sidx.as<uint16_t>() + (size_t)r0 * n, n, rows, c->pos.as<uint16_t>() + (size_t)r0 * n);
        CK(cudaGetLastError());
    }
    const int64_t mc = n * c->ncoarse;
    rb::coarse_kernel<<<(unsigned)((mc + 255) / 256), 256, 0, c->stream>>>(c->sdist.as<float>(), n, c->ncoarse,
                                                                          c->coarse.as<float>());
    CK(cudaGetLastError());
    c->cs1 = (c->ncoarse + 31) / 32;
    RET(c->coarse1.ensure((size_t)n * 32 * 4));
    rb::coarse1_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, c->stream>>>(c->coarse.as<float>(), n, c->ncoarse,
                                                                             c->cs1, c->coarse1.as<float>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int launch_units(riann_ctx *c, const float *frame, int H, int W, int C, float *unit, double *norms,
                 const float *prev_unit, double *tc)
{
    rb::UnitsParams U;
    U.frame = frame;
    U.H = H;
    U.W = W;
    U.C = C;
    U.pw = c->pw;
    U.ph = c->ph;
    U.gw = W - c->pw + 1;
    U.Q = (int64_t)U.gw * (H - c->ph + 1);
    U.dim = c->dim;
    U.unit = unit;
    U.norms = norms;
    U.prev_unit = prev_unit;
    U.tc = tc;
    if (U.Q <= 0) return 0;
    unsigned blocks = (unsigned)((U.Q + 127) / 128);
#ifndef RIANN_K1_TILE
#define RIANN_K1_TILE 1
#endif
    const int64_t k1_tiles = (int64_t)((U.gw + rb::K1_TW - 1) / rb::K1_TW) * ((H - c->ph + 1 + rb::K1_TH - 1) / rb::K1_TH);
    const unsigned k1_grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(k1_tiles, (int64_t)c->sms * 8));
    if (RIANN_K1_TILE && c->pw == 8 && c->ph == 8 && c->dim == 64 && C == 1) {
        rb::units_tile_kernel<64><<<k1_grid, 256, 0, c->stream>>>(U);
    } else if (RIANN_K1_TILE && c->pw == 8 && c->ph == 8 && c->dim == 192 && C == 3) {
        rb::units_tile_kernel<192><<<k1_grid, 256, 0, c->stream>>>(U);
    } else if (c->pw == 8 && c->ph == 8 && c->dim == 64) {
        const unsigned b = (unsigned)std::min<int64_t>((U.Q + 31) / 32, (int64_t)c->sms * 16);
        rb::units_warp_kernel<64><<<b, 256, 0, c->stream>>>(U);
    } else if (c->pw == 8 && c->ph == 8 && c->dim == 192) {
        const unsigned b = (unsigned)std::min<int64_t>((U.Q + 15) / 16, (int64_t)c->sms * 16);
        rb::units_warp_kernel<192><<<b, 256, 0, c->stream>>>(U);
    } else if (c->pw == 8 && c->ph == 8) {
        rb::units_kernel<8, 8><<<blocks, 128, 0, c->stream>>>(U);
    } else {
        rb::units_kernel<0, 0><<<blocks, 128, 0, c->stream>>>(U);
    }
    CK(cudaGetLastError());
    return 0;
}

int check_frame(riann_ctx *c, int H, int W, int C)
{
    if (C != c->C)
        return fail(RIANN_E_DIMENSION, "frame has %d channels, model expects %d", C, c->C);
    if (W < c->pw || H < c->ph)
        return fail(RIANN_E_DIMENSION, "frame %dx%d smaller than patch %dx%d", W, H, c->pw, c->ph);
    return 0;
}

// ---- host numpy RNG (init_field) ----
typedef unsigned __int128 u128;
const u128 HPCG_MULT = ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
struct HostPcg {
    u128 s, inc;
    int has;
    uint32_t buf;
};
uint32_t h_hash(uint32_t v, uint32_t &hc)
{
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    v ^= v >> 16;
    return v;
}
uint32_t h_mix(uint32_t x, uint32_t y)
{
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
}
void h_seed(HostPcg &g, const uint32_t *w, int nw)
{
    uint32_t pool[4], hc = 0x43b0d7e5u;
    for (int i = 0; i < 4; i++) pool[i] = h_hash(i < nw ? w[i] : 0u, hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = h_mix(pool[d], h_hash(pool[s], hc));
    for (int s = 4; s < nw; s++)
        for (int d = 0; d < 4; d++) pool[d] = h_mix(pool[d], h_hash(w[s], hc));
    uint32_t st[8], hb = 0x8b51f9ddu;
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= 0x58f38dedu;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    uint64_t w0 = st[0] | ((uint64_t)st[1] << 32), w1 = st[2] | ((uint64_t)st[3] << 32);
    uint64_t w2 = st[4] | ((uint64_t)st[5] << 32), w3 = st[6] | ((uint64_t)st[7] << 32);
    g.inc = ((((u128)w2 << 64) | w3) << 1) | 1u;
    g.s = g.inc;
    g.s += ((u128)w0 << 64) | w1;
    g.s = g.s * HPCG_MULT + g.inc;
    g.has = 0;
    g.buf = 0;
}
uint32_t h_next32(HostPcg &g)
{
    if (g.has) {
        g.has = 0;
        return g.buf;
    }
    g.s = g.s * HPCG_MULT + g.inc;
    uint64_t x = (uint64_t)(g.s >> 64) ^ (uint64_t)g.s;
    unsigned rot = (unsigned)(g.s >> 122);
    uint64_t v = (x >> rot) | (x << ((64u - rot) & 63u));
    g.has = 1;
    g.buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
}
uint64_t h_integers(HostPcg &g, uint64_t k)
{
    uint64_t rng = k - 1;
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFull) return h_next32(g);
    uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)h_next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (0xFFFFFFFFu - (uint32_t)rng) % excl;
        while (left < thr) {
            m = (uint64_t)h_next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return m >> 32;
}

double h_pairwise(const double *a, int64_t n)
{
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += a[i];
        return s;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) s += a[i];
        return s;
    }
    int64_t h = n / 2;
    h -= h % 8;
    return h_pairwise(a, h) + h_pairwise(a + h, n - h);
}

}  // namespace

// ===========================================================================
extern "C" {

int riann_abi_version(void) { return RIANN_ABI_VERSION; }
int riann_debug_checks(void)
{
#ifdef RIANN_BOUNDS
    return 1;
#else
    return 0;
#endif
}
const char *riann_last_error(void) { return g_err.c_str(); }

int riann_ctx_create(int device, riann_ctx **out)
{
    if (!out) return fail(RIANN_E_VALUE, "out is null");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(RIANN_E_VALUE, "device %d out of range (%d devices)", device, ndev);
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(RIANN_E_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);
    riann_ctx *c = new riann_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    c->smem_optin = (int)prop.sharedMemPerBlockOptin;
    // stream priorities: the frame path first, the side streams (K2 stragglers,
    // projection / temporal-change tree) fill idle SM slots
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
#ifndef RIANN_STREAM_PRIO
#define RIANN_STREAM_PRIO 1
#endif
    if (!RIANN_STREAM_PRIO) prio_lo = prio_hi = 0;
    cudaError_t e = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_lo);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_p0, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_heavy, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->stream3, cudaStreamNonBlocking, prio_lo);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_units, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_proj, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_tc, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        delete c;
        return fail(RIANN_E_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    if (c->err.ensure(64) || c->stats.ensure(64) || c->tc_sum.ensure(64) || c->small.ensure(64)) {
        delete c;
        return RIANN_E_CAPACITY;
    }
    *out = c;
    return 0;
}

int riann_ctx_destroy(riann_ctx *c)
{
    if (!c) return 0;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    DevBuf *bufs[] = {&c->refs, &c->refs16, &c->err16, &c->dmat, &c->pos, &c->coarse, &c->coarse1, &c->b_state, &c->b_pool,
                      &c->b_active[0], &c->b_active[1], &c->b_heavy, &c->b_counters, &c->b_counts, &c->b_starts,
                      &c->b_gdesc, &c->b_bits, &c->b_kept, &c->b_heavy2, &c->b_heavy3, &c->overflow2, &c->pca_T, &c->refs_pca16, &c->e16p, &c->sh_ptrs,
                      &c->units_pca, &c->e16max, &c->snap_idx, &c->snap_units, &c->sdist, &c->sidx, &c->frame, &c->units[0], &c->units[1], &c->prev,
                      &c->fld_idx[0], &c->fld_idx[1], &c->fld_dist, &c->tc, &c->tc_sum, &c->stats,
                      &c->err, &c->overflow, &c->keys, &c->kw, &c->koff, &c->q_rings, &c->q_evals,
                      &c->q_cand, &c->q_first, &c->q_scanned, &c->q_scanned_len, &c->small,
                      &c->tree.leaf_start, &c->tree.leaf_len, &c->tree.leaf_node, &c->tree.level_off,
                      &c->tree.inner, &c->tree.left, &c->tree.right, &c->tree.node_val, &c->x_B, &c->x_nr, &c->x_center, &c->x_scal,
                      &c->x_A, &c->x_nq, &c->x_cand, &c->x_lb, &c->x_ncand, &c->x_ub, &c->x_fb, &c->x_q,
                      &c->x_idx, &c->x_dist, &c->fx_frame, &c->fx_idx, &c->fx_pay, &c->fx_norm, &c->fx_out,
                      &c->fx_rgb, &c->pack};
    for (DevBuf *b : bufs) b->release();
    for (auto &kv : c->parked) kv.second.release();
    c->parked.clear();
    for (auto &a : c->ev_pending)
        for (auto e : a) cudaEventDestroy(e);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    cudaStreamSynchronize(c->stream2);
    cudaStreamSynchronize(c->stream3);
    cudaEventDestroy(c->ev_p0);
    cudaEventDestroy(c->ev_heavy);
    cudaEventDestroy(c->ev_units);
    cudaEventDestroy(c->ev_proj);
    cudaEventDestroy(c->ev_tc);
    cudaStreamDestroy(c->stream2);
    cudaStreamDestroy(c->stream3);
    cudaStreamDestroy(c->stream);
    delete c;
    return 0;
}

void *riann_ctx_stream(riann_ctx *c) { return c ? (void *)c->stream : nullptr; }

int riann_sync(riann_ctx *c)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    RET(c->use());
    CK(cudaStreamSynchronize(c->stream));
    return check_err(c);
}

uint64_t riann_ctx_device_bytes(riann_ctx *c) { return c ? c->bytes() : 0; }

int riann_ctx_set_path(riann_ctx *c, int path)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (path < 0 || path > 3)
        return fail(RIANN_E_VALUE, "path must be a mask of 1 (per-query frame kernel) and 2 (SIMT exact comparator)");
    c->bulk_disabled = (path & 1) != 0;
    c->exact_simt = (path & 2) != 0;
    return 0;
}

int riann_slot_select(riann_ctx *c, int slot)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (slot < 0) return fail(RIANN_E_VALUE, "slot must be >= 0, got %d", slot);
    if (slot == c->slot) return 0;
    RET(c->use());
    CK(cudaStreamSynchronize(c->stream));
    StreamState cur;
    c->swap_state(cur);  // active -> cur, active becomes empty
    c->parked[c->slot] = std::move(cur);
    auto it = c->parked.find(slot);
    if (it != c->parked.end()) {
        c->swap_state(it->second);
        c->parked.erase(it);
    }
    c->slot = slot;
    return 0;
}

int riann_slot_current(riann_ctx *c) { return c ? c->slot : -1; }

int riann_slot_free(riann_ctx *c, int slot)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    RET(c->use());
    CK(cudaStreamSynchronize(c->stream));
    if (slot == c->slot) {
        StreamState cur;
        c->swap_state(cur);
        cur.release();
        if (slot != 0) RET(riann_slot_select(c, 0));
        return 0;
    }
    auto it = c->parked.find(slot);
    if (it != c->parked.end()) {
        it->second.release();
        c->parked.erase(it);
    }
    return 0;
}

int riann_model_set_refs(riann_ctx *c, const float *refs, int64_t n, int dim, int pw, int ph, int channels,
                         int metric_id)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (metric_id != 0)
        return fail(RIANN_E_UNSUPPORTED, "metric id %d: only the Euclidean metric (id 0) has a GPU path", metric_id);
    if (n < 1) return fail(RIANN_E_VALUE, "need at least one reference, got n=%lld", (long long)n);
    if (n > 0x7fffffffLL) return fail(RIANN_E_CAPACITY, "n=%lld exceeds int32 indices", (long long)n);
    if (dim < 1 || pw < 1 || ph < 1 || channels < 1 || (int64_t)pw * ph * channels != dim)
        return fail(RIANN_E_DIMENSION, "dim %d != patch %dx%d x %d channels", dim, pw, ph, channels);
    RET(c->use());
    CK(cudaStreamSynchronize(c->stream));
    c->sdist.release();
    c->sidx.release();
    c->dmat.release();
    c->nshards = 0;
    c->own_rows = -1;
    c->pos.release();
    c->coarse.release();
    c->coarse1.release();
    c->tables = false;
    c->x_ready = false;
    RET(c->refs.ensure((size_t)n * dim * 4));
    CK(cudaMemcpyAsync(c->refs.p, refs, (size_t)n * dim * 4, cudaMemcpyHostToDevice, c->stream));
    RET(c->refs16.ensure((size_t)n * dim * 2));
    RET(c->err16.ensure((size_t)n * 4));
    rb::refs16_kernel<<<(unsigned)((n + 127) / 128), 128, 0, c->stream>>>(c->refs.as<float>(), n, dim,
                                                                          c->refs16.as<__half>(), c->err16.as<float>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    c->n = n;
    c->dim = dim;
    RET(build_pca(c, refs));
    c->pw = pw;
    c->ph = ph;
    c->C = channels;
    c->field_count = -1;
    c->have_prev_units = false;
    c->snap_valid = false;
    for (auto &kv : c->parked) {
        kv.second.field_count = -1;
        kv.second.have_prev_units = false;
        kv.second.snap_valid = false;
    }
    return 0;
}

int riann_model_set_tables(riann_ctx *c, const float *sd, const int32_t *si)
{
    RET(check_model(c, false));
    RET(c->use());
    const int64_t n = c->n;
    const size_t cnt = (size_t)n * n;
    c->idx16 = n <= 65536;
    RET(c->sdist.ensure(cnt * 4));
    RET(c->sidx.ensure(cnt * (c->idx16 ? 2 : 4)));
    // index-ordered distance rows only for n > 65,536 (rank rows serve K2 otherwise)
    if (c->idx16) c->dmat.release();
    else RET(c->dmat.ensure(cnt * 4));
    CK(cudaMemcpyAsync(c->sdist.p, sd, cnt * 4, cudaMemcpyHostToDevice, c->stream));
    // index rows in chunks through a staging buffer (narrowed to u16 when possible)
    const int64_t chunk_rows = std::max<int64_t>(1, (int64_t)((256ull << 20) / ((size_t)n * 4)));
    DevBuf stage;
    RET(stage.ensure((size_t)std::min<int64_t>(chunk_rows, n) * n * 4));
    for (int64_t r0 = 0; r0 < n; r0 += chunk_rows) {
        const int64_t rows = std::min<int64_t>(chunk_rows, n - r0);
        const size_t m = (size_t)rows * n;
        CK(cudaMemcpyAsync(stage.p, si + (size_t)r0 * n, m * 4, cudaMemcpyHostToDevice, c->stream));
        const unsigned blocks = (unsigned)((m + 255) / 256);
        if (c->idx16) {
            uint16_t *dst = c->sidx.as<uint16_t>() + (size_t)r0 * n;
            rb::narrow_u16_kernel<<<blocks, 256, 0, c->stream>>>(stage.as<int32_t>(), dst, (int64_t)m);
        } else {
            int32_t *dst = c->sidx.as<int32_t>() + (size_t)r0 * n;
            CK(cudaMemcpyAsync(dst, stage.p, m * 4, cudaMemcpyDeviceToDevice, c->stream));
            rb::dmat_scatter_kernel<int32_t><<<blocks, 256, 0, c->stream>>>(
                c->sdist.as<float>() + (size_t)r0 * n, dst, n, rows, c->dmat.as<float>() + (size_t)r0 * n);
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));
    }
    stage.release();
    RET(build_bulk_tables(c));
    c->nshards = 0;
    c->own_row0 = 0;
    c->own_rows = n;
    c->tables = true;
    return 0;
}

// K3 for table rows [row_lo, row_lo + nrows): sorted rows, index rows and the
// index-ordered distance rows, stored from row_lo on (a shard holds a row range)
int build_table_rows(riann_ctx *c, int64_t row_lo, int64_t nrows, bool want_dmat)
{
    const int64_t n = c->n;
    const size_t tcnt = (size_t)nrows * n;
    c->idx16 = n <= 65536;
    RET(c->sdist.ensure(tcnt * 4));
    RET(c->sidx.ensure(tcnt * (c->idx16 ? 2 : 4)));
    // index-ordered distance rows: only where the per-query kernel has no rank
    // rows to use instead (row shards, n > 65,536)
    if (want_dmat) RET(c->dmat.ensure(tcnt * 4));
    else c->dmat.release();
    // row batches bounded by ~1 GiB of unsorted keys+values
    int64_t rb_rows = (int64_t)((1ull << 30) / ((size_t)n * 8));
    if (rb_rows < 1) rb_rows = 1;
    if (rb_rows > n) rb_rows = n;
    if ((int64_t)rb_rows * n > 0x7fffffffLL) rb_rows = 0x7fffffffLL / n;
    RET(c->keys.ensure((size_t)rb_rows * n * 12));
    uint32_t *keys_in = c->keys.as<uint32_t>();
    int32_t *vals_in = reinterpret_cast<int32_t *>(keys_in + (size_t)rb_rows * n);
    int32_t *vals_out = vals_in + (size_t)rb_rows * n;
    // segment offsets r*n
    std::vector<int> offs(rb_rows + 1);
    for (int64_t r = 0; r <= rb_rows; r++) offs[r] = (int)(r * n);
    DevBuf d_off;
    RET(d_off.ensure(offs.size() * 4));
    CK(cudaMemcpy(d_off.p, offs.data(), offs.size() * 4, cudaMemcpyHostToDevice));
    size_t temp_bytes = 0;
    CK(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp_bytes, keys_in, (uint32_t *)nullptr, vals_in,
                                                 (int32_t *)nullptr, (int)(rb_rows * n), (int)rb_rows,
                                                 d_off.as<int>(), d_off.as<int>() + 1, 0, 32, c->stream));
    DevBuf temp;
    RET(temp.ensure(temp_bytes));
    const int64_t row_hi = row_lo + nrows;
    for (int64_t r0 = row_lo; r0 < row_hi; r0 += rb_rows) {
        const int64_t rows = (r0 + rb_rows <= row_hi) ? rb_rows : row_hi - r0;
        const size_t ro = (size_t)(r0 - row_lo) * n;  // storage offset of row r0
        const unsigned blocks = (unsigned)std::min<int64_t>((rows + 7) / 8, (int64_t)c->sms * 8);
        switch (c->dim) {
        case 16: rb::table_keys_kernel<16><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), n, c->dim, r0, rows, keys_in, vals_in); break;
        case 64: rb::table_keys_kernel<64><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), n, c->dim, r0, rows, keys_in, vals_in); break;
        case 192: rb::table_keys_kernel<192><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), n, c->dim, r0, rows, keys_in, vals_in); break;
        default: rb::table_keys_kernel<0><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), n, c->dim, r0, rows, keys_in, vals_in); break;
        }
        CK(cudaGetLastError());
        // index-ordered distances are the unsorted keys
        if (want_dmat)
            CK(cudaMemcpyAsync(c->dmat.as<float>() + ro, keys_in, (size_t)rows * n * 4,
                               cudaMemcpyDeviceToDevice, c->stream));
        uint32_t *kout = reinterpret_cast<uint32_t *>(c->sdist.as<float>() + ro);
        int32_t *vout = c->idx16 ? vals_out : c->sidx.as<int32_t>() + ro;
        CK(cub::DeviceSegmentedRadixSort::SortPairs(temp.p, temp_bytes, keys_in, kout, vals_in, vout,
                                                     (int)(rows * n), (int)rows, d_off.as<int>(),
                                                     d_off.as<int>() + 1, 0, 32, c->stream));
        rb::self_first_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, c->stream>>>(kout, vout, n, r0, rows);
        CK(cudaGetLastError());
        if (c->idx16) {
            rb::narrow_u16_kernel<<<(unsigned)((rows * n + 255) / 256), 256, 0, c->stream>>>(
                vout, c->sidx.as<uint16_t>() + ro, rows * n);
            CK(cudaGetLastError());
        }
    }
    CK(cudaStreamSynchronize(c->stream));
    temp.release();
    d_off.release();
    c->keys.release();
    return 0;
}

int riann_model_build_tables(riann_ctx *c)
{
    RET(check_model(c, false));
    RET(c->use());
    RET(build_table_rows(c, 0, c->n, c->n > 65536));
    RET(build_bulk_tables(c));
    c->nshards = 0;
    c->own_row0 = 0;
    c->own_rows = c->n;
    c->tables = true;
    return 0;
}

int riann_model_build_table_rows(riann_ctx *c, int64_t row0, int64_t rows)
{
    RET(check_model(c, false));
    if (row0 < 0 || rows < 1 || row0 + rows > c->n)
        return fail(RIANN_E_INDEX, "rows [%lld, %lld) out of range for %lld references", (long long)row0,
                    (long long)(row0 + rows), (long long)c->n);
    RET(c->use());
    c->pos.release();
    c->coarse.release();
    c->coarse1.release();
    RET(build_table_rows(c, row0, rows, true));  // shards: K2 reads dmat rows
    c->nshards = 0;
    c->own_row0 = row0;
    c->own_rows = rows;
    c->tables = row0 == 0 && rows == c->n;
    if (c->tables) RET(build_bulk_tables(c));
    return 0;
}

int riann_model_table_ptrs(riann_ctx *c, void **sd, void **si, void **dm, int64_t *row0, int64_t *rows)
{
    RET(check_model(c, false));
    if (c->own_rows < 0 || !c->sdist.p) return fail(RIANN_E_STATE, "context holds no table rows");
    if (sd) *sd = c->sdist.p;
    if (si) *si = c->sidx.p;
    if (dm) *dm = c->dmat.p;
    if (row0) *row0 = c->own_row0;
    if (rows) *rows = c->own_rows;
    return 0;
}

int riann_model_detach_shards(riann_ctx *c)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    RET(c->use());
    CK(cudaStreamSynchronize(c->stream));
    if (c->nshards > 0) {
        c->nshards = 0;
        c->tables = false;
        c->field_count = -1;
        c->sh_ptrs.release();
    }
    return 0;
}

int riann_model_attach_shards(riann_ctx *c, int nshards, int64_t shard_rows, void *const *sd, void *const *si,
                              void *const *dm)
{
    RET(check_model(c, false));
    if (nshards < 1 || nshards > 64 || shard_rows < 1 || (int64_t)nshards * shard_rows < c->n ||
        (int64_t)(nshards - 1) * shard_rows >= c->n)
        return fail(RIANN_E_VALUE, "%d shards of %lld rows do not tile %lld rows", nshards, (long long)shard_rows,
                    (long long)c->n);
    RET(c->use());
    // peer access to shards on other GPUs (NVLink peer loads)
    for (int s = 0; s < nshards; s++) {
        for (void *ptr : {sd[s], si[s], dm[s]}) {
            if (!ptr) return fail(RIANN_E_VALUE, "shard %d has a null table pointer", s);
            cudaPointerAttributes at;
            CK(cudaPointerGetAttributes(&at, ptr));
            if (at.type != cudaMemoryTypeDevice) return fail(RIANN_E_VALUE, "shard %d is not device memory", s);
            if (at.device != c->device) {
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, c->device, at.device));
                if (!ok) return fail(RIANN_E_UNSUPPORTED, "device %d cannot access peer %d", c->device, at.device);
                const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
            }
        }
    }
    std::vector<const void *> ptrs;
    for (int s = 0; s < nshards; s++) ptrs.push_back(sd[s]);
    for (int s = 0; s < nshards; s++) ptrs.push_back(si[s]);
    for (int s = 0; s < nshards; s++) ptrs.push_back(dm[s]);
    RET(c->sh_ptrs.ensure(ptrs.size() * sizeof(void *)));
    CK(cudaMemcpy(c->sh_ptrs.p, ptrs.data(), ptrs.size() * sizeof(void *), cudaMemcpyHostToDevice));
    c->nshards = nshards;
    c->shard_rows = shard_rows;
    c->idx16 = c->n <= 65536;
    c->tables = true;
    c->field_count = -1;
    return 0;
}

int riann_model_get_tables(riann_ctx *c, int64_t row0, int64_t rows, float *sd, int32_t *si)
{
    RET(check_model(c, false));
    if (c->nshards > 0) return fail(RIANN_E_UNSUPPORTED, "tables are attached shards: read them from their owners");
    if (c->own_rows < 0) return fail(RIANN_E_STATE, "model has no sorted tables");
    if (row0 < c->own_row0 || rows < 0 || row0 + rows > c->own_row0 + c->own_rows)
        return fail(RIANN_E_INDEX, "rows out of range");
    RET(c->use());
    const int64_t n = c->n;
    const size_t off = (size_t)(row0 - c->own_row0) * n, cnt = (size_t)rows * n;
    if (sd) CK(cudaMemcpyAsync(sd, c->sdist.as<float>() + off, cnt * 4, cudaMemcpyDeviceToHost, c->stream));
    if (si) {
        if (!c->idx16) {
            CK(cudaMemcpyAsync(si, c->sidx.as<int32_t>() + off, cnt * 4, cudaMemcpyDeviceToHost, c->stream));
        } else {
            const int64_t chunk = std::max<int64_t>(1, (int64_t)((256ull << 20) / ((size_t)n * 4)));
            DevBuf stage;
            RET(stage.ensure((size_t)std::min<int64_t>(chunk, rows) * n * 4));
            for (int64_t r = 0; r < rows; r += chunk) {
                const int64_t m = std::min<int64_t>(chunk, rows - r) * n;
                rb::widen_u16_kernel<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(
                    c->sidx.as<uint16_t>() + off + (size_t)r * n, stage.as<int32_t>(), m);
                CK(cudaGetLastError());
                CK(cudaMemcpyAsync(si + (size_t)r * n, stage.p, (size_t)m * 4, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
            }
        }
    }
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_set_prev_units(riann_ctx *c, const float *units, int64_t rows, int dim)
{
    RET(check_model(c, false));
    if (dim != c->dim) return fail(RIANN_E_DIMENSION, "prev_unit dim %d != model dim %d", dim, c->dim);
    RET(c->use());
    const int slot = c->cur_units ^ 1;
    RET(c->units[slot].ensure((size_t)rows * dim * 4));
    CK(cudaMemcpyAsync(c->units[slot].p, units, (size_t)rows * dim * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->have_prev_units = true;
    c->prev_units_rows = rows;
    return 0;
}

int riann_process_frame(riann_ctx *c, const float *frame, int H, int W, int C, int gy0, const int32_t *prev_idx,
                        uint64_t seed, uint32_t t, int L, double alpha, int max_rings, unsigned flags,
                        int32_t *out_idx, double *out_dist, riann_frame_stats *stats)
{
    RET(check_model(c, true));
    RET(check_frame(c, H, W, C));
    if (L < 1) return fail(RIANN_E_VALUE, "L must be >= 1, got %d", L);
    if (!(alpha > 0.0 && alpha < 1.0)) return fail(RIANN_E_VALUE, "alpha must lie in (0, 1), got %g", alpha);
    if (max_rings < 1) return fail(RIANN_E_VALUE, "max_rings must be >= 1, got %d", max_rings);
    if (gy0 < 0) return fail(RIANN_E_VALUE, "negative band offset");
    RET(c->use());
    const bool dev = (flags & RIANN_F_DEVICE_PTRS) != 0;
    const int gw = W - c->pw + 1, gh = H - c->ph + 1;
    const int64_t Q = (int64_t)gw * gh;
    const size_t fbytes = (size_t)H * W * C * 4;
    const float *d_frame = frame;
    if (!dev) {
        RET(c->frame.ensure(fbytes));
        CK(cudaMemcpyAsync(c->frame.p, frame, fbytes, cudaMemcpyHostToDevice, c->stream));
        d_frame = c->frame.as<float>();
    }
    // previous field
    const int32_t *d_prev = nullptr;
    const int in_slot = c->cur_fld, out_slot = c->cur_fld ^ 1;
    if (prev_idx) {
        if (dev) {
            d_prev = prev_idx;
        } else {
            RET(c->fld_idx[in_slot].ensure((size_t)Q * 4));
            CK(cudaMemcpyAsync(c->fld_idx[in_slot].p, prev_idx, (size_t)Q * 4, cudaMemcpyHostToDevice, c->stream));
            d_prev = c->fld_idx[in_slot].as<int32_t>();
        }
    } else {
        if (c->field_count != Q)
            return fail(RIANN_E_STATE, "no device-resident field of %lld positions (have %lld)", (long long)Q,
                        (long long)c->field_count);
        d_prev = c->fld_idx[in_slot].as<int32_t>();
    }
    int32_t *d_idx = nullptr;
    double *d_dist = nullptr;
    if (dev && out_idx && out_dist) {
        d_idx = out_idx;
        d_dist = out_dist;
    } else {
        RET(c->fld_idx[out_slot].ensure((size_t)Q * 4));
        RET(c->fld_dist.ensure((size_t)Q * 8));
        d_idx = c->fld_idx[out_slot].as<int32_t>();
        d_dist = c->fld_dist.as<double>();
    }
    // K1: units (+ temporal change per position)
    const bool temporal = (flags & RIANN_F_TEMPORAL) != 0;
    if (temporal && (!c->have_prev_units || c->prev_units_rows != Q))
        return fail(RIANN_E_DIMENSION, "prev_unit rows %lld do not match %lld positions",
                    (long long)(c->have_prev_units ? c->prev_units_rows : 0), (long long)Q);
    const int us = c->cur_units;
    RET(c->units[us].ensure((size_t)Q * c->dim * 4));
    if (temporal) RET(c->tc.ensure((size_t)Q * 8));
    std::array<cudaEvent_t, 4> evs = {nullptr, nullptr, nullptr, nullptr};
    if (c->timing) {
        for (auto &e : evs) e = c->ev();
        CK(cudaEventRecord(evs[0], c->stream));
    }
    c->launches += 1;
    tmark(c, PH_UNITS);
    RET(launch_units(c, d_frame, H, W, C, c->units[us].as<float>(), nullptr,
                     temporal ? c->units[us ^ 1].as<float>() : nullptr, temporal ? c->tc.as<double>() : nullptr));
    // K2: queries
    CK(cudaMemsetAsync(c->stats.p, 0, 64, c->stream));
    CK(cudaMemsetAsync(c->err.p, 0, 4, c->stream));
    rb::QueryParams P;
    memset(&P, 0, sizeof P);
    P.refs = c->refs.as<float>();
    P.sdist = c->sdist.as<float>();
    P.sidx = c->sidx.p;
    P.n = c->n;
    P.dim = c->dim;
    P.units = c->units[us].as<float>();
    P.prev = d_prev;
    P.Q = Q;
    P.seed_lo = (uint32_t)seed;
    P.seed_hi = (uint32_t)(seed >> 32);
    P.seed_nw = (seed >> 32) ? 2 : 1;
    P.gw = gw;
    P.gy0 = gy0;
    P.t = t;
    P.L = L;
    P.alpha = alpha;
    P.max_rings = max_rings;
    P.out_idx = d_idx;
    P.out_dist = d_dist;
    P.stats = c->stats.as<unsigned long long>();
    P.err = c->err.as<int>();
    if (c->timing) CK(cudaEventRecord(evs[1], c->stream));
    // temporal-change reduction: needs only K1's per-position values, so it
    // runs on the third stream alongside the query path
    const bool tree = temporal && Q > 0;
    if (tree) {
        CK(cudaEventRecord(c->ev_tc, c->stream));
        CK(cudaStreamWaitEvent(c->stream3, c->ev_tc, 0));
        RET(c->tree.build(Q));
        rb::PwTreeParams T;
        T.vals = c->tc.as<double>();
        T.nleaves = c->tree.nleaves;
        T.leaf_start = c->tree.leaf_start.as<int64_t>();
        T.leaf_len = c->tree.leaf_len.as<int32_t>();
        T.leaf_node = c->tree.leaf_node.as<int32_t>();
        T.nlevels = c->tree.nlevels;
        T.level_off = c->tree.level_off.as<int32_t>();
        T.inner_node = c->tree.inner.as<int32_t>();
        T.left = c->tree.left.as<int32_t>();
        T.right = c->tree.right.as<int32_t>();
        T.node_val = c->tree.node_val.as<double>();
        T.out = c->tc_sum.as<double>();
        rb::pw_tree_kernel<<<1, 1024, 0, c->stream3>>>(T);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->ev_tc, c->stream3));
        c->launches += 1;
    }
    if (Q > 0) {
        tmark(c, PH_QUERY);
        RET(launch_query(c, P));
        c->launches += 1;
    }
    tmark(c, -1);
    if (c->timing) CK(cudaEventRecord(evs[2], c->stream));
    if (tree) CK(cudaStreamWaitEvent(c->stream, c->ev_tc, 0));
    if (c->timing) {
        CK(cudaEventRecord(evs[3], c->stream));
        c->ev_pending.push_back(evs);
        c->marks_pending.push_back(std::move(c->marks));
        c->marks.clear();
    }
    if (!dev) {
        if (out_idx) CK(cudaMemcpyAsync(out_idx, d_idx, (size_t)Q * 4, cudaMemcpyDeviceToHost, c->stream));
        if (out_dist) CK(cudaMemcpyAsync(out_dist, d_dist, (size_t)Q * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    if (!(dev && d_idx == out_idx)) {
        c->cur_fld = out_slot;
        c->field_count = Q;
    } else {
        c->field_count = -1;
    }
    if (flags & RIANN_F_KEEP_UNITS) {
        c->cur_units ^= 1;
        c->have_prev_units = true;
        c->prev_units_rows = Q;
    }
    if ((flags & RIANN_F_ASYNC) && dev) return 0;
    unsigned long long hs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    double tcv = 0.0;
    CK(cudaMemcpyAsync(hs, c->stats.p, 64, cudaMemcpyDeviceToHost, c->stream));
    if (temporal && Q > 0) CK(cudaMemcpyAsync(&tcv, c->tc_sum.p, 8, cudaMemcpyDeviceToHost, c->stream));
    RET(check_err(c));
    if (stats) {
        stats->total_rings = hs[0];
        stats->total_distance_evals = hs[1];
        stats->sum_cand_final = hs[2];
        stats->sum_first_ring = hs[3];
        stats->queries = (uint64_t)Q;
        stats->temporal_change = tcv;
        stats->sum_ring_tests = hs[4];
        stats->sum_exact_evals = hs[5];
        stats->queries_fallback = hs[6];
    }
    return 0;
}

int riann_timing_enable(riann_ctx *c, int on)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    RET(c->use());
    CK(cudaStreamSynchronize(c->stream));
    for (auto &a : c->ev_pending)
        for (auto e : a) c->ev_pool.push_back(e);
    c->ev_pending.clear();
    for (auto &f : c->marks_pending)
        for (auto &m : f) c->ev_pool.push_back(m.second);
    c->marks_pending.clear();
    for (auto &m : c->marks) c->ev_pool.push_back(m.second);
    c->marks.clear();
    for (double &x : c->t_phase) x = 0.0;
    c->t_phase_frames.clear();
    c->timing = on != 0;
    c->t_ms[0] = c->t_ms[1] = c->t_ms[2] = 0.0;
    c->t_frames = 0;
    c->launches = 0;
    return 0;
}

int riann_timing_read(riann_ctx *c, double *ms3, uint64_t *frames, uint64_t *launches)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    RET(c->use());
    CK(cudaStreamSynchronize(c->stream));
    for (auto &a : c->ev_pending) {
        for (int k = 0; k < 3; k++) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, a[k], a[k + 1]));
            c->t_ms[k] += ms;
        }
        for (auto e : a) c->ev_pool.push_back(e);
        c->t_frames++;
    }
    c->ev_pending.clear();
    for (auto &f : c->marks_pending) {
        // the stretch between mark i and mark i+1 belongs to mark i's phase
        std::array<double, RIANN_NPHASES> fr{};
        for (size_t i = 0; i + 1 < f.size(); i++) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, f[i].second, f[i + 1].second));
            if (f[i].first >= 0) {
                c->t_phase[f[i].first] += ms;
                fr[f[i].first] += ms;
            }
        }
        c->t_phase_frames.push_back(fr);
        for (auto &m : f) c->ev_pool.push_back(m.second);
    }
    c->marks_pending.clear();
    if (ms3)
        for (int k = 0; k < 3; k++) ms3[k] = c->t_ms[k];
    if (frames) *frames = c->t_frames;
    if (launches) *launches = c->launches;
    return 0;
}

int riann_timing_phases(riann_ctx *c, double *ms, int nphases)
{
    RET(riann_timing_read(c, nullptr, nullptr, nullptr));
    for (int k = 0; k < nphases && k < RIANN_NPHASES; k++) ms[k] = c->t_phase[k];
    return 0;
}

int riann_timing_phases_frame(riann_ctx *c, int64_t frame, double *ms, int nphases)
{
    RET(riann_timing_read(c, nullptr, nullptr, nullptr));
    const int64_t nf = (int64_t)c->t_phase_frames.size();
    if (frame < 0) frame += nf;
    if (frame < 0 || frame >= nf) return fail(RIANN_E_INDEX, "timed frame %lld of %lld", (long long)frame, (long long)nf);
    for (int k = 0; k < nphases && k < RIANN_NPHASES; k++) ms[k] = c->t_phase_frames[(size_t)frame][k];
    return 0;
}

const char *riann_phase_name(int k) { return (k >= 0 && k < RIANN_NPHASES) ? kPhaseNames[k] : nullptr; }

int riann_state_save(riann_ctx *c)
{
    RET(check_model(c, true));
    if (c->field_count < 0) return fail(RIANN_E_STATE, "no device-resident field to save");
    RET(c->use());
    const int64_t Q = c->field_count;
    RET(c->snap_idx.ensure((size_t)Q * 4));
    CK(cudaMemcpyAsync(c->snap_idx.p, c->fld_idx[c->cur_fld].p, (size_t)Q * 4, cudaMemcpyDeviceToDevice, c->stream));
    c->snap_have_units = c->have_prev_units;
    c->snap_units_rows = c->prev_units_rows;
    if (c->have_prev_units) {
        const size_t ub = (size_t)c->prev_units_rows * c->dim * 4;
        RET(c->snap_units.ensure(ub));
        CK(cudaMemcpyAsync(c->snap_units.p, c->units[c->cur_units ^ 1].p, ub, cudaMemcpyDeviceToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    c->snap_field = Q;
    c->snap_valid = true;
    return 0;
}

int riann_state_restore(riann_ctx *c)
{
    RET(check_model(c, true));
    if (!c->snap_valid) return fail(RIANN_E_STATE, "no saved state");
    RET(c->use());
    const int64_t Q = c->snap_field;
    RET(c->fld_idx[c->cur_fld].ensure((size_t)Q * 4));
    CK(cudaMemcpyAsync(c->fld_idx[c->cur_fld].p, c->snap_idx.p, (size_t)Q * 4, cudaMemcpyDeviceToDevice, c->stream));
    c->field_count = Q;
    c->have_prev_units = c->snap_have_units;
    c->prev_units_rows = c->snap_units_rows;
    if (c->snap_have_units) {
        const size_t ub = (size_t)c->snap_units_rows * c->dim * 4;
        RET(c->units[c->cur_units ^ 1].ensure(ub));
        CK(cudaMemcpyAsync(c->units[c->cur_units ^ 1].p, c->snap_units.p, ub, cudaMemcpyDeviceToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_field_get(riann_ctx *c, int32_t *idx, double *dist, int64_t count)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (c->field_count != count) return fail(RIANN_E_STATE, "no device field of %lld positions", (long long)count);
    RET(c->use());
    if (idx) CK(cudaMemcpyAsync(idx, c->fld_idx[c->cur_fld].p, (size_t)count * 4, cudaMemcpyDeviceToHost, c->stream));
    if (dist) CK(cudaMemcpyAsync(dist, c->fld_dist.p, (size_t)count * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_tc_get(riann_ctx *c, double *out, int64_t count, unsigned flags)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (count < 0 || (size_t)count * 8 > c->tc.cap)
        return fail(RIANN_E_STATE, "no per-position temporal change of %lld positions", (long long)count);
    RET(c->use());
    const bool dev = (flags & RIANN_F_DEVICE_PTRS) != 0;
    CK(cudaMemcpyAsync(out, c->tc.p, (size_t)count * 8, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       c->stream));
    if (!dev) CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_frame_units(riann_ctx *c, const float *frame, int H, int W, int C, float *unit, double *norms)
{
    RET(check_model(c, false));
    RET(check_frame(c, H, W, C));
    RET(c->use());
    const int64_t Q = (int64_t)(W - c->pw + 1) * (H - c->ph + 1);
    const size_t fbytes = (size_t)H * W * C * 4;
    RET(c->frame.ensure(fbytes));
    CK(cudaMemcpyAsync(c->frame.p, frame, fbytes, cudaMemcpyHostToDevice, c->stream));
    DevBuf u, nr;
    RET(u.ensure((size_t)Q * c->dim * 4));
    RET(nr.ensure((size_t)Q * 8));
    RET(launch_units(c, c->frame.as<float>(), H, W, C, u.as<float>(), nr.as<double>(), nullptr, nullptr));
    if (unit) CK(cudaMemcpyAsync(unit, u.p, (size_t)Q * c->dim * 4, cudaMemcpyDeviceToHost, c->stream));
    if (norms) CK(cudaMemcpyAsync(norms, nr.p, (size_t)Q * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    u.release();
    nr.release();
    return 0;
}

}  // extern "C"

namespace {

template <class T>
int normalize_rows_t(riann_ctx *c, const T *values, int64_t m, int dim, float *unit, double *norms)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (dim < 1 || m < 0) return fail(RIANN_E_DIMENSION, "bad shape (%lld, %d)", (long long)m, dim);
    if (m == 0) return 0;
    RET(c->use());
    DevBuf v, u, nr;
    RET(v.ensure((size_t)m * dim * sizeof(T)));
    RET(u.ensure((size_t)m * dim * 4));
    RET(nr.ensure((size_t)m * 8));
    CK(cudaMemcpyAsync(v.p, values, (size_t)m * dim * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    rb::normalize_rows_kernel<T><<<(unsigned)((m + 127) / 128), 128, 0, c->stream>>>(v.as<T>(), m, dim, u.as<float>(),
                                                                                     nr.as<double>());
    CK(cudaGetLastError());
    if (unit) CK(cudaMemcpyAsync(unit, u.p, (size_t)m * dim * 4, cudaMemcpyDeviceToHost, c->stream));
    if (norms) CK(cudaMemcpyAsync(norms, nr.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

template <class T>
int one_to_many_t(riann_ctx *c, const T *q, const T *rows, int64_t k, int dim, double *out)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (dim < 1 || k < 0) return fail(RIANN_E_DIMENSION, "bad shape (%lld, %d)", (long long)k, dim);
    if (k == 0) return 0;
    RET(c->use());
    DevBuf dq, dr, dout;
    RET(dq.ensure((size_t)dim * sizeof(T)));
    RET(dr.ensure((size_t)k * dim * sizeof(T)));
    RET(dout.ensure((size_t)k * 8));
    CK(cudaMemcpyAsync(dq.p, q, (size_t)dim * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dr.p, rows, (size_t)k * dim * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    rb::one_to_many_kernel<T><<<(unsigned)((k + 127) / 128), 128, 0, c->stream>>>(dq.as<T>(), dr.as<T>(), k, dim,
                                                                                  dout.as<double>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout.p, (size_t)k * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

}  // namespace

extern "C" {

int riann_normalize_rows(riann_ctx *c, const float *values, int64_t m, int dim, float *unit, double *norms)
{
    return normalize_rows_t<float>(c, values, m, dim, unit, norms);
}

int riann_normalize_rows_f64(riann_ctx *c, const double *values, int64_t m, int dim, float *unit, double *norms)
{
    return normalize_rows_t<double>(c, values, m, dim, unit, norms);
}

int riann_one_to_many(riann_ctx *c, const float *q, const float *rows, int64_t k, int dim, double *out)
{
    return one_to_many_t<float>(c, q, rows, k, dim, out);
}

int riann_one_to_many_f64(riann_ctx *c, const double *q, const double *rows, int64_t k, int dim, double *out)
{
    return one_to_many_t<double>(c, q, rows, k, dim, out);
}

int riann_extract_patches(riann_ctx *c, const float *frame, int H, int W, int C, int pw, int ph, int stride,
                          float *out)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (pw < 1 || ph < 1) return fail(RIANN_E_DIMENSION, "patch size must be positive, got (%d, %d)", pw, ph);
    if (stride < 1) return fail(RIANN_E_DIMENSION, "stride must be >= 1, got %d", stride);
    if (W < pw || H < ph) return fail(RIANN_E_DIMENSION, "frame %dx%d smaller than patch %dx%d", W, H, pw, ph);
    RET(c->use());
    const int gw = (W - pw) / stride + 1, gh = (H - ph) / stride + 1;
    const int64_t Q = (int64_t)gw * gh;
    const size_t fbytes = (size_t)H * W * C * 4, obytes = (size_t)Q * pw * ph * C * 4;
    DevBuf f, o;
    RET(f.ensure(fbytes));
    RET(o.ensure(obytes));
    CK(cudaMemcpyAsync(f.p, frame, fbytes, cudaMemcpyHostToDevice, c->stream));
    rb::extract_kernel<<<(unsigned)((Q + 127) / 128), 128, 0, c->stream>>>(f.as<float>(), W, C, pw, ph, stride, gw, Q,
                                                                           o.as<float>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, o.p, obytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_ring_candidates(riann_ctx *c, int64_t anchor, double d, double eps, int64_t *lo, int64_t *hi, int32_t *out)
{
    if (c && c->nshards > 0) return fail(RIANN_E_UNSUPPORTED, "ring_candidates on attached shards");
    RET(check_model(c, true));
    if (anchor < 0 || anchor >= c->n)
        return fail(RIANN_E_INDEX, "anchor %lld out of range for %lld references", (long long)anchor, (long long)c->n);
    if (d < 0 || eps < 0) return fail(RIANN_E_VALUE, "ring radius and width must be nonnegative");
    RET(c->use());
    rb::ring_window_kernel<<<1, 32, 0, c->stream>>>(c->sdist.as<float>() + (size_t)anchor * c->n, c->n, d - eps,
                                                   d + eps, c->small.as<int64_t>());
    CK(cudaGetLastError());
    int64_t h[2];
    CK(cudaMemcpyAsync(h, c->small.p, 16, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *lo = h[0];
    *hi = h[1];
    if (out && h[1] > h[0]) {
        const size_t m = (size_t)(h[1] - h[0]);
        if (c->idx16) {
            std::vector<uint16_t> tmp(m);
            CK(cudaMemcpy(tmp.data(), c->sidx.as<uint16_t>() + (size_t)anchor * c->n + h[0], m * 2,
                          cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < m; i++) out[i] = tmp[i];
        } else {
            CK(cudaMemcpy(out, c->sidx.as<int32_t>() + (size_t)anchor * c->n + h[0], m * 4, cudaMemcpyDeviceToHost));
        }
    }
    return 0;
}

int riann_query_batch(riann_ctx *c, const float *queries, const int32_t *prev, const uint32_t *key_words,
                      const int64_t *key_off, int64_t m, int L, double alpha, int max_rings, int32_t *out_idx,
                      double *out_dist, int32_t *out_rings, int64_t *out_evals, int64_t *out_cand,
                      int64_t *out_first, int32_t *scanned, int64_t *scanned_len)
{
    RET(check_model(c, true));
    if (L < 1) return fail(RIANN_E_VALUE, "L must be >= 1, got %d", L);
    if (!(alpha > 0.0 && alpha < 1.0)) return fail(RIANN_E_VALUE, "alpha must lie in (0, 1), got %g", alpha);
    if (max_rings < 1) return fail(RIANN_E_VALUE, "max_rings must be >= 1, got %d", max_rings);
    if (m <= 0) return 0;
    for (int64_t i = 0; i < m; i++) {
        if (prev[i] < 0 || prev[i] >= c->n)
            return fail(RIANN_E_INDEX, "prev_index %d out of range for %lld references", prev[i], (long long)c->n);
        if (key_off[i + 1] - key_off[i] > 16 || key_off[i + 1] < key_off[i])
            return fail(RIANN_E_UNSUPPORTED, "rng key of %lld words (max 16)", (long long)(key_off[i + 1] - key_off[i]));
    }
    RET(c->use());
    const int64_t nk = key_off[m];
    DevBuf dq, dp, di, dd;
    RET(dq.ensure((size_t)m * c->dim * 4));
    RET(dp.ensure((size_t)m * 4));
    RET(di.ensure((size_t)m * 4));
    RET(dd.ensure((size_t)m * 8));
    RET(c->kw.ensure((size_t)(nk + 1) * 4));
    RET(c->koff.ensure((size_t)(m + 1) * 8));
    CK(cudaMemcpyAsync(dq.p, queries, (size_t)m * c->dim * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dp.p, prev, (size_t)m * 4, cudaMemcpyHostToDevice, c->stream));
    if (nk) CK(cudaMemcpyAsync(c->kw.p, key_words, (size_t)nk * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->koff.p, key_off, (size_t)(m + 1) * 8, cudaMemcpyHostToDevice, c->stream));
    RET(c->q_rings.ensure((size_t)m * 4));
    RET(c->q_evals.ensure((size_t)m * 8));
    RET(c->q_cand.ensure((size_t)m * 8));
    RET(c->q_first.ensure((size_t)m * 8));
    RET(c->q_scanned_len.ensure((size_t)m * 8));
    if (scanned) RET(c->q_scanned.ensure((size_t)m * (c->n + 1) * 4));
    CK(cudaMemsetAsync(c->err.p, 0, 4, c->stream));
    rb::QueryParams P;
    memset(&P, 0, sizeof P);
    P.refs = c->refs.as<float>();
    P.sdist = c->sdist.as<float>();
    P.sidx = c->sidx.p;
    P.n = c->n;
    P.dim = c->dim;
    P.units = dq.as<float>();
    P.prev = dp.as<int32_t>();
    P.Q = m;
    P.key_words = c->kw.as<uint32_t>();
    P.key_off = c->koff.as<int64_t>();
    P.gw = 1;
    P.L = L;
    P.alpha = alpha;
    P.max_rings = max_rings;
    P.out_idx = di.as<int32_t>();
    P.out_dist = dd.as<double>();
    P.out_rings = c->q_rings.as<int32_t>();
    P.out_evals = c->q_evals.as<int64_t>();
    P.out_cand = c->q_cand.as<int64_t>();
    P.out_first = c->q_first.as<int64_t>();
    P.scanned = scanned ? c->q_scanned.as<int32_t>() : nullptr;
    P.scanned_len = c->q_scanned_len.as<int64_t>();
    P.stats = nullptr;
    P.err = c->err.as<int>();
    RET(launch_query(c, P));
    if (out_idx) CK(cudaMemcpyAsync(out_idx, di.p, (size_t)m * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_dist) CK(cudaMemcpyAsync(out_dist, dd.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (out_rings) CK(cudaMemcpyAsync(out_rings, c->q_rings.p, (size_t)m * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_evals) CK(cudaMemcpyAsync(out_evals, c->q_evals.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (out_cand) CK(cudaMemcpyAsync(out_cand, c->q_cand.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (out_first) CK(cudaMemcpyAsync(out_first, c->q_first.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (scanned_len) CK(cudaMemcpyAsync(scanned_len, c->q_scanned_len.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (scanned) CK(cudaMemcpyAsync(scanned, c->q_scanned.p, (size_t)m * (c->n + 1) * 4, cudaMemcpyDeviceToHost, c->stream));
    RET(check_err(c));
    return 0;
}

}  // extern "C"

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D fp16 operand (rows, kcols), K-major, 64 x box_rows boxes with the 128-byte swizzle
int encode_operand(CUtensorMap *map, const void *base, int64_t rows, int kcols, int box_rows)
{
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) return fail(RIANN_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)p;
    }
    cuuint64_t dims[2] = {(cuuint64_t)kcols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kcols * 2};
    cuuint32_t box[2] = {(cuuint32_t)rb::tc::BK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(RIANN_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return 0;
}

// Relative screen error E: |d2_est - d^2| <= E (||q'||^2 + ||r'||^2) + E_abs with q', r' the
// centred rows (exact_scal_kernel computes E_abs):
//   fp16 operand rounding (unit roundoff u = 2^-11, normal range after the power-of-two
//     scaling):  |q^.r^ - q.r| <= (2u + u^2) ||q|| ||r||, doubled for d^2
//   fp32 accumulation of K = D exact products: 2K * 2^-23 * sum|q_i r_i| (4x the
//     round-to-nearest gamma_K, for adders that truncate), doubled for d^2
//   centring, norm rounding and the float arithmetic of the bounds: < 64 * 2^-24
// using 2 ||q|| ||r|| <= ||q||^2 + ||r||^2.
float exact_eps(int K)
{
    const double u = std::ldexp(1.0, -11);
    return (float)((2 * u + u * u) * 1.01 + 2.1 * K * std::ldexp(1.0, -23) + 64 * std::ldexp(1.0, -24));
}

// fallback list (m int32) then the counters [fallbacks i32, pad, checked u64], 16-byte aligned
size_t fb_counters_off(int64_t m) { return ((size_t)m * 4 + 15) & ~(size_t)15; }

bool exact_tc_ok(const riann_ctx *c) { return !c->exact_simt && (c->dim == 64 || c->dim == 192); }

template <int D>
int exact_tc_run(riann_ctx *c, const float *dq, int64_t m, int32_t *didx, double *ddist)
{
    namespace T = rb::tc;
    constexpr int KB = D / T::BK;
    const int64_t n = c->n;
    const unsigned eblocks = (unsigned)c->sms * 8;
    const float E = exact_eps(D);
    // x_center: [center f32 x D | pad to 8 | acc f64 x D]; x_scal: [Scal | maxr u32 | maxq u32]
    RET(c->x_scal.ensure(64));
    T::Scal *scal = c->x_scal.as<T::Scal>();
    unsigned *maxr = reinterpret_cast<unsigned *>(c->x_scal.as<char>() + 16);
    unsigned *maxq = maxr + 1;
    const float *center = c->x_center.as<float>();
    if (!c->x_ready) {
        RET(c->x_B.ensure((size_t)n * D * 2));
        RET(c->x_nr.ensure((size_t)n * 8 + ((size_t)(n + 31) / 32) * 4));
        RET(c->x_center.ensure((size_t)D * 16 + 16));
        center = c->x_center.as<float>();
        double *cacc = reinterpret_cast<double *>(c->x_center.as<char>() + (((size_t)D * 4 + 15) & ~(size_t)15));
        CK(cudaMemsetAsync(cacc, 0, (size_t)D * 8, c->stream));
        CK(cudaMemsetAsync(maxr, 0, 4, c->stream));
        T::center_sum_kernel<<<(unsigned)((n + 1023) / 1024), D, 0, c->stream>>>(c->refs.as<float>(), n, D, cacc);
        T::center_fin_kernel<<<1, D, 0, c->stream>>>(cacc, n, D, c->x_center.as<float>());
        T::absmax_kernel<<<eblocks, 256, 0, c->stream>>>(c->refs.as<float>(), center, n, D, maxr);
        T::split_kernel<<<eblocks, 256, 0, c->stream>>>(c->refs.as<float>(), center, n, D, maxr,
                                                        c->x_B.as<__half>());
        T::norm2_kernel<<<eblocks, 256, 0, c->stream>>>(c->refs.as<float>(), center, n, D, E, nullptr,
                                                        c->x_nr.as<float>(), c->x_nr.as<float>() + n);
        T::chunk_slack_kernel<<<eblocks, 256, 0, c->stream>>>(c->x_nr.as<float>(), c->x_nr.as<float>() + n, n,
                                                              c->x_nr.as<float>() + 2 * n);
        CK(cudaGetLastError());
        c->x_ready = true;
    }
    RET(c->x_A.ensure((size_t)m * D * 2));
    RET(c->x_nq.ensure((size_t)m * 4));
    RET(c->x_cand.ensure((size_t)m * 2 * T::NCAND * 4));
    RET(c->x_lb.ensure((size_t)m * 2 * T::NCAND * 4));
    RET(c->x_ncand.ensure((size_t)m * 8));
    RET(c->x_ub.ensure((size_t)m * 8));
    RET(c->x_fb.ensure(fb_counters_off(m) + 64));
    CK(cudaMemsetAsync(maxq, 0, 4, c->stream));
    T::absmax_kernel<<<eblocks, 256, 0, c->stream>>>(dq, center, m, D, maxq);
    T::split_kernel<<<eblocks, 256, 0, c->stream>>>(dq, center, m, D, maxq, c->x_A.as<__half>());
    T::norm2_kernel<<<eblocks, 256, 0, c->stream>>>(dq, center, m, D, E, c->x_nq.as<float>(), nullptr, nullptr);
    T::exact_scal_kernel<<<1, 1, 0, c->stream>>>(maxq, maxr, D, E, scal);
    CK(cudaGetLastError());
    CUtensorMap mapA, mapB;
    RET(encode_operand(&mapA, c->x_A.p, m, D, T::BM));
    RET(encode_operand(&mapB, c->x_B.p, n, D, T::BN));
    T::ExactParams P{};
    P.nq = c->x_nq.as<float>();
    P.nrU = c->x_nr.as<float>();
    P.nrL = c->x_nr.as<float>() + n;
    P.dlt = c->x_nr.as<float>() + 2 * n;
    P.scal = scal;
    P.m = m;
    P.n = n;
    P.kblocks = KB;
    P.stages = T::stages_for(KB);
    P.cand = c->x_cand.as<int32_t>();
    P.cand_lb = c->x_lb.as<float>();
    P.ncand = c->x_ncand.as<int32_t>();
    P.best_ub = c->x_ub.as<float>();
    const int smem = T::smem_bytes(KB);
    CK(cudaFuncSetAttribute(T::exact_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    T::exact_tc_kernel<<<(unsigned)((m + T::BM - 1) / T::BM), T::THREADS, smem, c->stream>>>(mapA, mapB, P);
    CK(cudaGetLastError());
    int32_t *nfb = reinterpret_cast<int32_t *>(c->x_fb.as<char>() + fb_counters_off(m));
    unsigned long long *nchk = reinterpret_cast<unsigned long long *>(c->x_fb.as<char>() + fb_counters_off(m) + 8);
    CK(cudaMemsetAsync(nfb, 0, 16, c->stream));
    const unsigned rblocks = (unsigned)std::min<int64_t>((m + 7) / 8, (int64_t)c->sms * 16);
    T::exact_recheck_kernel<D><<<rblocks, 256, 0, c->stream>>>(c->refs.as<float>(), n, dq, m, P.cand, P.cand_lb,
                                                               P.ncand, P.best_ub, didx, ddist, c->x_fb.as<int32_t>(),
                                                               nfb, nchk);
    T::exact_list_kernel<D><<<(unsigned)c->sms * 8, 256, 0, c->stream>>>(c->refs.as<float>(), n, dq,
                                                                         c->x_fb.as<int32_t>(), nfb, didx, ddist);
    CK(cudaGetLastError());
    c->launches += 8;
    return 0;
}

// K4 on device buffers: tensor-core screen + exact re-check, or the SIMT scan
int exact_run(riann_ctx *c, const float *dq, int64_t m, int32_t *didx, double *ddist)
{
    if (exact_tc_ok(c)) {
        if (c->dim == 64) return exact_tc_run<64>(c, dq, m, didx, ddist);
        return exact_tc_run<192>(c, dq, m, didx, ddist);
    }
    const unsigned blocks = (unsigned)((m + 7) / 8 < (int64_t)c->sms * 8 ? (m + 7) / 8 : (int64_t)c->sms * 8);
    switch (c->dim) {
    case 16: rb::exact_nn_kernel<16><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), c->n, c->dim, dq, m, didx, ddist); break;
    case 64: rb::exact_nn_kernel<64><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), c->n, c->dim, dq, m, didx, ddist); break;
    case 192: rb::exact_nn_kernel<192><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), c->n, c->dim, dq, m, didx, ddist); break;
    default: rb::exact_nn_kernel<0><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), c->n, c->dim, dq, m, didx, ddist); break;
    }
    CK(cudaGetLastError());
    c->launches += 1;
    return 0;
}

}  // namespace

extern "C" {

int riann_exact_nn_device(riann_ctx *c, const float *queries, int64_t m, int32_t *out_idx, double *out_dist,
                          uint64_t *stats)
{
    RET(check_model(c, false));
    if (m < 0) return fail(RIANN_E_VALUE, "negative query count");
    RET(c->use());
    if (m > 0) RET(exact_run(c, queries, m, out_idx, out_dist));
    if (stats) {
        stats[0] = stats[1] = 0;
        if (m > 0 && exact_tc_ok(c)) {
            int32_t h[4];
            CK(cudaMemcpyAsync(h, c->x_fb.as<char>() + fb_counters_off(m), 16, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            unsigned long long chk;
            std::memcpy(&chk, h + 2, 8);
            stats[0] = chk;
            stats[1] = (uint64_t)h[0];
        }
    }
    return 0;
}

int riann_exact_nn_batch(riann_ctx *c, const float *queries, int64_t m, int32_t *out_idx, double *out_dist)
{
    RET(check_model(c, false));
    if (m <= 0) return 0;
    RET(c->use());
    RET(c->x_q.ensure((size_t)m * c->dim * 4));
    RET(c->x_idx.ensure((size_t)m * 4));
    RET(c->x_dist.ensure((size_t)m * 8));
    CK(cudaMemcpyAsync(c->x_q.p, queries, (size_t)m * c->dim * 4, cudaMemcpyHostToDevice, c->stream));
    RET(exact_run(c, c->x_q.as<float>(), m, c->x_idx.as<int32_t>(), c->x_dist.as<double>()));
    CK(cudaMemcpyAsync(out_idx, c->x_idx.p, (size_t)m * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(out_dist, c->x_dist.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_exact_field(riann_ctx *c, const float *frame, int H, int W, int C, int32_t *out_idx, double *out_dist)
{
    RET(check_model(c, false));
    RET(check_frame(c, H, W, C));
    RET(c->use());
    const int64_t Q = (int64_t)(W - c->pw + 1) * (H - c->ph + 1);
    const size_t fbytes = (size_t)H * W * C * 4;
    RET(c->frame.ensure(fbytes));
    CK(cudaMemcpyAsync(c->frame.p, frame, fbytes, cudaMemcpyHostToDevice, c->stream));
    RET(c->x_q.ensure((size_t)Q * c->dim * 4));
    RET(c->x_idx.ensure((size_t)Q * 4));
    RET(c->x_dist.ensure((size_t)Q * 8));
    RET(launch_units(c, c->frame.as<float>(), H, W, C, c->x_q.as<float>(), nullptr, nullptr, nullptr));
    // bounded launches (config 4: 8.25 M queries x 262,144 references)
    const int64_t chunk = (int64_t)1 << 20;
    for (int64_t q0 = 0; q0 < Q; q0 += chunk) {
        const int64_t m = std::min(chunk, Q - q0);
        RET(exact_run(c, c->x_q.as<float>() + q0 * c->dim, m, c->x_idx.as<int32_t>() + q0, c->x_dist.as<double>() + q0));
    }
    CK(cudaMemcpyAsync(out_idx, c->x_idx.p, (size_t)Q * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(out_dist, c->x_dist.p, (size_t)Q * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_field_pack(riann_ctx *c, void *payload, int64_t count)
{
    if (!c) return fail(RIANN_E_STATE, "null context");
    if (c->field_count != count) return fail(RIANN_E_STATE, "no device field of %lld positions", (long long)count);
    RET(c->use());
    if (count <= 0) return 0;
    RET(c->pack.ensure((size_t)count * 8));
    rb::pack_field_kernel<<<(unsigned)((count + 255) / 256), 256, 0, c->stream>>>(
        c->fld_idx[c->cur_fld].as<int32_t>(), c->fld_dist.as<double>(), count, c->pack.as<uint32_t>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(payload, c->pack.p, (size_t)count * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_apply_effect(riann_ctx *c, const float *frame, int H, int W, const int32_t *idx, const float *payloads,
                       int64_t n_payloads, int payload_dim, int kind, float *out_planes, uint8_t *out_rgb)
{
    RET(check_model(c, false));
    if (kind < 0 || kind > 2) return fail(RIANN_E_VALUE, "unknown payload kind %d", kind);
    if (c->C != 1 && !(c->pw * c->ph == c->dim))
        return fail(RIANN_E_DIMENSION, "effects need a single-plane model (transforms.py:217-218)");
    const int pw = c->pw, ph = c->ph, pp = pw * ph;
    if (H < ph || W < pw) return fail(RIANN_E_DIMENSION, "frame %dx%d smaller than patch %dx%d", W, H, pw, ph);
    const int planes = kind == rb::FX_CHROMA ? 2 : 1;
    if (kind == rb::FX_RECONSTRUCTION && !payloads) {
        n_payloads = c->n;
        payload_dim = c->dim;
    }
    if (n_payloads != c->n)
        return fail(RIANN_E_DIMENSION, "table holds %lld payloads for a model of %lld references",
                    (long long)n_payloads, (long long)c->n);
    if (payload_dim != planes * pp)
        return fail(RIANN_E_DIMENSION, "payloads must be (n, %d), got width %d", planes * pp, payload_dim);
    const int gw = W - pw + 1, gh = H - ph + 1;
    const int64_t Q = (int64_t)gw * gh, P = (int64_t)H * W;
    RET(c->use());
    RET(c->fx_frame.ensure((size_t)P * 4));
    CK(cudaMemcpyAsync(c->fx_frame.p, frame, (size_t)P * 4, cudaMemcpyHostToDevice, c->stream));
    const int32_t *didx;
    if (idx) {
        RET(c->fx_idx.ensure((size_t)Q * 4));
        CK(cudaMemcpyAsync(c->fx_idx.p, idx, (size_t)Q * 4, cudaMemcpyHostToDevice, c->stream));
        didx = c->fx_idx.as<int32_t>();
    } else {
        if (c->field_count != Q)
            return fail(RIANN_E_STATE, "no device field of %lld positions", (long long)Q);
        didx = c->fld_idx[c->cur_fld].as<int32_t>();
    }
    const float *dpay = c->refs.as<float>();
    if (payloads) {
        RET(c->fx_pay.ensure((size_t)n_payloads * payload_dim * 4));
        CK(cudaMemcpyAsync(c->fx_pay.p, payloads, (size_t)n_payloads * payload_dim * 4, cudaMemcpyHostToDevice,
                           c->stream));
        dpay = c->fx_pay.as<float>();
    }
    rb::BlendParams B{};
    B.frame = c->fx_frame.as<float>();
    B.H = H;
    B.W = W;
    B.pw = pw;
    B.ph = ph;
    B.gw = gw;
    B.gh = gh;
    B.idx = didx;
    B.payloads = dpay;
    B.planes = planes;
    B.kind = kind;
    if (kind == rb::FX_RECONSTRUCTION) {
        RET(c->fx_norm.ensure((size_t)Q * 8));
        if (pw == 8 && ph == 8 && c->dim == 64) {  // warp-cooperative K1, norms only
            RET(launch_units(c, B.frame, H, W, 1, nullptr, c->fx_norm.as<double>(), nullptr, nullptr));
        } else {
            rb::effect_norms_kernel<<<(unsigned)((Q + 127) / 128), 128, 0, c->stream>>>(
                B.frame, H, W, pw, ph, gw, Q, c->fx_norm.as<double>());
            CK(cudaGetLastError());
        }
        B.norms = c->fx_norm.as<double>();
    }
    if (out_planes) {
        RET(c->fx_out.ensure((size_t)planes * P * 4));
        B.out = c->fx_out.as<float>();
    }
    if (kind == rb::FX_CHROMA && out_rgb) {
        RET(c->fx_rgb.ensure((size_t)P * 3));
        B.rgb = c->fx_rgb.as<uint8_t>();
    }
    if (pw <= 16) {
        const size_t sm = (size_t)planes * rb::BY * (rb::BX + pw - 1) * pw * 4;
        CK(cudaFuncSetAttribute(rb::blend_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        const dim3 grid((unsigned)((W + rb::BX - 1) / rb::BX), (unsigned)((H + rb::BY - 1) / rb::BY));
        rb::blend_tiled_kernel<<<grid, rb::BX * rb::BY, sm, c->stream>>>(B);
    } else {
        rb::blend_kernel<<<(unsigned)((P + 255) / 256), 256, 0, c->stream>>>(B);
    }
    CK(cudaGetLastError());
    if (out_planes) CK(cudaMemcpyAsync(out_planes, B.out, (size_t)planes * P * 4, cudaMemcpyDeviceToHost, c->stream));
    if (B.rgb) CK(cudaMemcpyAsync(out_rgb, B.rgb, (size_t)P * 3, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->launches += 2;
    return 0;
}

int riann_pair_dist(riann_ctx *c, const int32_t *ia, const int32_t *ib, const float *u, int64_t m, double *out_ab,
                    double *out_au)
{
    RET(check_model(c, false));
    if (m < 0) return fail(RIANN_E_VALUE, "negative pair count");
    if (m == 0) return 0;
    RET(c->use());
    DevBuf di, dj, du, dab, dau;
    RET(di.ensure((size_t)m * 4));
    RET(dj.ensure((size_t)m * 4));
    RET(dab.ensure((size_t)m * 8));
    CK(cudaMemcpyAsync(di.p, ia, (size_t)m * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dj.p, ib, (size_t)m * 4, cudaMemcpyHostToDevice, c->stream));
    if (u) {
        RET(du.ensure((size_t)m * c->dim * 4));
        RET(dau.ensure((size_t)m * 8));
        CK(cudaMemcpyAsync(du.p, u, (size_t)m * c->dim * 4, cudaMemcpyHostToDevice, c->stream));
    }
    const unsigned blocks = (unsigned)std::min<int64_t>((m + 7) / 8, (int64_t)c->sms * 16);
    const float *dup = u ? du.as<float>() : nullptr;
    switch (c->dim) {
    case 16: rb::pair_dist_kernel<16><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), di.as<int32_t>(), dj.as<int32_t>(), dup, m, c->dim, dab.as<double>(), dau.as<double>()); break;
    case 64: rb::pair_dist_kernel<64><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), di.as<int32_t>(), dj.as<int32_t>(), dup, m, c->dim, dab.as<double>(), dau.as<double>()); break;
    case 192: rb::pair_dist_kernel<192><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), di.as<int32_t>(), dj.as<int32_t>(), dup, m, c->dim, dab.as<double>(), dau.as<double>()); break;
    default: rb::pair_dist_kernel<0><<<blocks, 256, 0, c->stream>>>(c->refs.as<float>(), di.as<int32_t>(), dj.as<int32_t>(), dup, m, c->dim, dab.as<double>(), dau.as<double>()); break;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_ab, dab.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (u && out_au) CK(cudaMemcpyAsync(out_au, dau.p, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int riann_init_field(int gw, int gh, int64_t n, const uint32_t *seed_words, int nwords, int32_t *out)
{
    if (n < 1) return fail(RIANN_E_VALUE, "need at least one reference, got n=%lld", (long long)n);
    if (gw < 1 || gh < 1) return fail(RIANN_E_VALUE, "empty grid %dx%d", gw, gh);
    if (n > 0x7fffffffLL) return fail(RIANN_E_VALUE, "n too large for int32 indices");
    HostPcg g;
    h_seed(g, seed_words, nwords);
    const int64_t total = (int64_t)gw * gh;
    for (int64_t i = 0; i < total; i++) out[i] = (int32_t)h_integers(g, (uint64_t)n);
    return 0;
}

double riann_pairwise_sum(const double *a, int64_t n) { return h_pairwise(a, n); }

}  // extern "C"
