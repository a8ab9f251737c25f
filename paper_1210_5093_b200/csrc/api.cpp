// api.cpp -- the C ABI of include/dfa.h: handle, device tables, scratch,
// launch orchestration.  See include/dfa.h for the contract.
#include "../../include/dfa.h"
#include "kernels.cuh"
#include "prep.h"

#include <cuda.h>  // CUtensorMap (types only: the encoder is taken from the driver at run time)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

using namespace dfa;

#ifndef DFA_SHAPE_PCT
// grouped split: keep at least this share of the estimated sub-chunk count when rounding it to a
// multiple of the warp group (Random: 23 sub-chunks per chunk in groups of 1 fill 147 of 148 SMs with
// 20 warps; 22 in groups of 2 -- the 95 % rule of round 1 -- left the same 20 warps on 141 SMs with
// longer sub-chunks: lanes kernel 0.1256 vs 0.1317 ms, step 0.1422 vs 0.1448 ms)
#define DFA_SHAPE_PCT 97
#endif

namespace {

// Bumped whenever a scratch buffer is (re)allocated or a composition tree's
// arrival counters are reset: a captured CUDA graph holds raw scratch pointers
// and counter residues, so its replay key includes this generation.
std::atomic<uint64_t> g_scratch_gen{0};

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        g_scratch_gen++;
        if (p) { cudaFree(p); p = nullptr; cap = 0; }
        size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

struct HostPinned {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        if (p) { cudaFreeHost(p); p = nullptr; cap = 0; }
        cudaError_t e = cudaMallocHost(&p, std::max<size_t>(bytes, 64));
        if (e == cudaSuccess) cap = std::max<size_t>(bytes, 64);
        return e;
    }
    void release() { if (p) cudaFreeHost(p); p = nullptr; cap = 0; }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};


} // namespace

struct dfa_handle {
    Prep prep;
    bool device_ready = false;
    int device = 0, sms = 0, optin_smem = 0;
    DevBuf tables;
    DevTables T{};
    uint32_t c_num = 1, c_den = 1;
    // options
    int convergence = 1, profile = 0, threads = 512, threads_auto = 1;
    uint32_t tree_fanin_cap = 32;
    uint32_t walk_fanin = 8;
    int64_t subchunk_target = 0;
    // scratch
    DevBuf status, sfin, dom_of, surv, surv_n, surv_pos, amap;
    DevBuf lvlA, domA, counters, bounds, input, fold_rows, fold_doms, ticket, leaf_rows, leaf_dom, plan_bounds;
    DevBuf cta_start, leaf_rows2, leaf_dom2;
    DevBuf node_nv, node_fl, rep_full, clinks;  // factored composition (long rows behind the converge stage)
    int warp_compose = 1;
    int factored = 1;             // DFA_OPT_FACTORED
    int lookahead2 = 1;           // DFA_OPT_LOOKAHEAD2
    int tma_input = 0;            // DFA_OPT_TMA_INPUT (measured slower than register loads: DESIGN.md section 11)
    DevBuf tmap;                  // device copy of the input's tensor map (TMA input staging)
    CUtensorMap tmap_host;        // its host image (persistent: the upload reads it)
    uint64_t tmap_base = 0, tmap_rows = 0;
    DevBuf dom2;                  // two-symbol initial sets + sizes (converge stage)
    int fused_tail = 0;           // DFA_OPT_FUSED_TAIL (measured slower than compose8: DESIGN.md)
    DevBuf part_rows, part_doms, chunk_cnt;
    std::vector<uint64_t> plan_key;
    // CUDA graph of a repeated dfa_chunk_maps call
    int use_graphs = 1;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    std::vector<uint64_t> graph_key, graph_pending;
    uint32_t graph_kernels = 0;
    struct { uint32_t m0, m, g_log; int threads; } plan_split_c{};
    int fold_in_tree = 0;
    int max_lanes = kLanes;       // lanes per thread (DFA_OPT_MAX_LANES, 1..8)
    uint32_t sticky_avail = 0;    // the DFA has sticky states (upload)
    int sticky_parking = 1;       // DFA_OPT_STICKY_PARKING
    int count_work = 0;           // DFA_OPT_COUNT_WORK
    DevBuf work;                  // [2] u64 lane-step counters (converge, lanes)
    bool work_pending = false;
    uint32_t work_calls = 0;
    std::vector<uint64_t> tree_sig;
    HostPinned h_status, h_bounds;
    cudaEvent_t staging_done = nullptr;
    bool staging_pending = false;
    cudaStream_t last_stream = nullptr;
    // stats / profiling: event pairs around each kernel section, accumulated
    // over calls until dfa_get_stats reads (and resets) them
    dfa_stats stats{};
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Rec { int section; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    int open_section = -1;
    cudaEvent_t open_event = nullptr;
    std::vector<Rec> graph_recs;
    // dfa_match_host pipeline: pieces copied on copy_stream, matched on the caller's
    uint64_t host_piece = 32ull << 20;
    int early_exit = 1;
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> hm_ev;  // [2 * pieces]: copied, done
    DevBuf hm_rows, hm_bounds, hm_la, hm_final;
    HostPinned h_hm;
    // reporting rows of the last run (batch outputs read them)
    const uint16_t *rep_rows = nullptr;
    uint32_t rep_rs = 8;
    DevBuf batch_bounds, batch_kidx;
    HostPinned h_batch;
};

namespace {

dfa_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return DFA_OK;
    if (e == cudaErrorMemoryAllocation) return DFA_ERR_OOM;
    return DFA_ERR_CUDA;
}

thread_local char g_detail[512] = "";

dfa_status cuda_fail(cudaError_t e, const char *expr, int line) {
    std::snprintf(g_detail, sizeof g_detail, "%s (%s) at api.cpp:%d: %s", cudaGetErrorName(e),
                  cudaGetErrorString(e), line, expr);
    return cuda_status(e);
}

#define CK(expr)                                                         \
    do {                                                                 \
        cudaError_t _e = (expr);                                         \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr, __LINE__);    \
    } while (0)

uint32_t gcd32(uint32_t a, uint32_t b) {
    while (b) { uint32_t t = a % b; a = b; b = t; }
    return a;
}

// ----- device table upload --------------------------------------------------
dfa_status upload(dfa_handle *h) {
    Prep &p = h->prep;
    CK(cudaGetDevice(&h->device));
    CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->device));
    CK(cudaDeviceGetAttribute(&h->optin_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));

    const uint32_t nq = p.nq, nc = p.nclass, imax = p.imax, imu = p.imax_user_stride;
    std::vector<uint32_t> image = p.image;
    while (image.size() % 4) image.push_back(0);
    const uint32_t dls = (imax + 7) & ~7u;  // dom_list row stride = rs (16-byte rows)
    std::vector<uint16_t> dom_list((size_t)(nc + 1) * dls, kNone), dom_size(nc + 1, 0);
    std::vector<uint16_t> rank((size_t)(nc + 1) * nq, kNone);
    std::vector<uint8_t> rank8(imax < 255 ? (size_t)(nc + 1) * nq : 0, 0xFF);
    for (uint32_t c = 0; c <= nc; c++) {
        dom_size[c] = (uint16_t)p.dom[c].size();
        for (uint32_t j = 0; j < p.dom[c].size(); j++) {
            dom_list[(size_t)c * dls + j] = p.dom[c][j];
            rank[(size_t)c * nq + p.dom[c][j]] = (uint16_t)j;
            if (!rank8.empty()) rank8[(size_t)c * nq + p.dom[c][j]] = (uint8_t)j;
        }
    }
    const uint32_t rs = (imax + 7) & ~7u;
    std::vector<uint16_t> xlat((size_t)nc * imu, 0), dom_user_size(nc, 0), ixlat((size_t)nc * rs, kNone);
    for (uint32_t c = 0; c < nc; c++) {
        dom_user_size[c] = (uint16_t)p.dom_user[c].size();
        for (uint32_t j = 0; j < p.xlat[c].size(); j++) {
            xlat[(size_t)c * imu + j] = p.xlat[c][j];
            ixlat[(size_t)c * rs + p.xlat[c][j]] = (uint16_t)j;
        }
    }
    const uint32_t bw = ((nq + 31) / 32 + 3) & ~3u;
    std::vector<uint32_t> dead(bw, 0), absorb(bw, 0), accept(bw, 0), dead_user(bw, 0), sticky(bw, 0);
    {
        // universal kill bytes: every state goes to Z; sticky: not in Z, not absorbing,
        // and every other byte keeps the state (see checkpoint() in kernels.cu)
        std::vector<uint8_t> kill(256, 1);
        for (uint32_t b = 0; b < 256; b++)
            for (uint32_t q = 0; q < nq && kill[b]; q++)
                if (!p.dead[p.full[(size_t)q * 256 + b]]) kill[b] = 0;
        for (uint32_t q = 0; q < nq; q++) {
            if (p.dead[q] || p.absorbing[q]) continue;
            bool st = true;
            for (uint32_t b = 0; b < 256 && st; b++)
                if (!kill[b] && p.full[(size_t)q * 256 + b] != q) st = false;
            if (st) sticky[q >> 5] |= 1u << (q & 31);
        }
    }
    for (uint32_t q = 0; q < nq; q++) {
        if (p.dead[q]) dead[q >> 5] |= 1u << (q & 31);
        if (q < p.nq_user && p.dead_user[q]) dead_user[q >> 5] |= 1u << (q & 31);
        if (p.absorbing[q]) absorb[q >> 5] |= 1u << (q & 31);
        if (p.accepting[q]) accept[q >> 5] |= 1u << (q & 31);
    }
    // one allocation, 256-byte aligned sections
    struct Sec { const void *src; size_t bytes; size_t off; };
    std::vector<Sec> secs = {
        {image.data(), image.size() * 4, 0},
        {p.full.data(), p.full.size() * 2, 0},
        {p.byte_class.data(), 256, 0},
        {dom_list.data(), dom_list.size() * 2, 0},
        {dom_size.data(), dom_size.size() * 2, 0},
        {rank.data(), rank.size() * 2, 0},
        {dead.data(), dead.size() * 4, 0},
        {absorb.data(), absorb.size() * 4, 0},
        {accept.data(), accept.size() * 4, 0},
        {xlat.data(), xlat.size() * 2, 0},
        {dom_user_size.data(), dom_user_size.size() * 2, 0},
        {rank8.data(), rank8.size(), 0},
        {ixlat.data(), ixlat.size() * 2, 0},
        {dead_user.data(), dead_user.size() * 4, 0},
        {sticky.data(), sticky.size() * 4, 0},
    };
    size_t total = 0;
    for (auto &s : secs) { s.off = total; total += (s.bytes + 255) & ~size_t(255); }
    CK(h->tables.ensure(total));
    std::vector<uint8_t> blob(total, 0);
    for (auto &s : secs) if (s.bytes) std::memcpy(blob.data() + s.off, s.src, s.bytes);
    CK(cudaMemcpy(h->tables.p, blob.data(), total, cudaMemcpyHostToDevice));
    auto at = [&](int i) { return reinterpret_cast<const uint8_t *>(h->tables.p) + secs[i].off; };
    DevTables &T = h->T;
    T.image = reinterpret_cast<const uint32_t *>(at(0));
    T.image_words = p.mode == kGlobalU16 ? 0 : (uint32_t)image.size();
    T.gtable = reinterpret_cast<const uint16_t *>(at(1));
    T.byte_class = at(2);
    T.dom_list = reinterpret_cast<const uint16_t *>(at(3));
    T.dom_size = reinterpret_cast<const uint16_t *>(at(4));
    T.rank = reinterpret_cast<const uint16_t *>(at(5));
    T.dead_bits = reinterpret_cast<const uint32_t *>(at(6));
    T.absorb_bits = reinterpret_cast<const uint32_t *>(at(7));
    T.accept_bits = reinterpret_cast<const uint32_t *>(at(8));
    T.xlat = reinterpret_cast<const uint16_t *>(at(9));
    T.dom_user_size = reinterpret_cast<const uint16_t *>(at(10));
    T.rank8 = rank8.empty() ? nullptr : at(11);
    T.ixlat = reinterpret_cast<const uint16_t *>(at(12));
    T.dead_user_bits = reinterpret_cast<const uint32_t *>(at(13));
    T.sticky_bits = reinterpret_cast<const uint32_t *>(at(14));
    // two-symbol initial sets for the converge stage (Eq.istatesm, r = 2): delta(I_c1, c2) \ Z
    // as (state, rank in I_c2) pairs; skipped for small I_max (no converge stage), the Alg.2
    // ablation and tables over 128 MiB
    T.dom2 = nullptr;
    T.dom2_size = nullptr;
    T.dom2_stride = 0;
    if (imax > (uint32_t)kLanes && !p.full_domain && nq <= 0x7F00u &&
        (size_t)nc * nc * imax * 4 <= (size_t)512 << 20) {  // (no point in building what cannot fit)
        std::vector<std::vector<uint32_t>> sets((size_t)nc * nc);
        std::vector<uint8_t> mark(nq);
        uint32_t smax = 0;
        for (uint32_t c1 = 0; c1 < nc; c1++)
            for (uint32_t c2 = 0; c2 < nc; c2++) {
                std::fill(mark.begin(), mark.end(), 0);
                const uint32_t b = p.class_rep[c2];
                for (uint16_t q : p.dom[c1]) mark[p.full[(size_t)q * 256 + b]] = 1;
                auto &v = sets[(size_t)c1 * nc + c2];
                for (uint32_t j = 0; j < p.dom[c2].size(); j++)  // ascending states = ascending ranks
                    if (mark[p.dom[c2][j]]) v.push_back((uint32_t)p.dom[c2][j] | (j << 16));
                smax = std::max<uint32_t>(smax, (uint32_t)v.size());
            }
        const size_t entries = (size_t)nc * nc * smax;
        if (smax && entries * 4 <= (size_t)128 << 20) {
            std::vector<uint32_t> flat(entries, 0xFFFFFFFFu);
            std::vector<uint16_t> sz((size_t)nc * nc);
            for (size_t i = 0; i < sets.size(); i++) {
                sz[i] = (uint16_t)sets[i].size();
                std::copy(sets[i].begin(), sets[i].end(), flat.begin() + i * smax);
            }
            const size_t szoff = (entries * 4 + 255) & ~size_t(255);
            CK(h->dom2.ensure(szoff + sz.size() * 2));
            CK(cudaMemcpy(h->dom2.p, flat.data(), entries * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(static_cast<uint8_t *>(h->dom2.p) + szoff, sz.data(), sz.size() * 2, cudaMemcpyHostToDevice));
            T.dom2 = h->dom2.as<uint32_t>();
            T.dom2_size = reinterpret_cast<const uint16_t *>(static_cast<uint8_t *>(h->dom2.p) + szoff);
            T.dom2_stride = smax;
        }
    }
    T.has_sticky = 0;
    for (uint32_t w : sticky) T.has_sticky |= w != 0;
    h->sticky_avail = T.has_sticky;
    T.has_sticky = h->sticky_avail && h->sticky_parking;
    T.nq_user = p.nq_user;
    T.ns = p.ns;
    T.nq = nq;
    T.nclass = nc;
    T.start_dom = p.start_dom;
    T.imax = imax;
    T.imax_user = imu;
    T.rs = (imax + 7) & ~7u;
    T.has_dead = 0;
    T.has_absorb = 0;
    for (uint32_t q = 0; q < nq; q++) T.has_dead |= p.dead[q];
    for (uint32_t q = 0; q < nq; q++) T.has_absorb |= p.absorbing[q];
    T.stride = p.stride;
    T.win_base = p.win_base;
    T.win_w = p.win_w;
    T.mode = p.mode;
    T.q0 = p.q0;
    T.poison = p.poison == kNone ? 0xFFFFFFFFu : p.poison;
    if ((int)(T.image_words * 4 + bw * 4) > h->optin_smem) return DFA_ERR_INTERNAL;
    CK(setup_kernel_attributes(T));
    CK(h->status.ensure(sizeof(DevStatus)));
    CK(h->h_status.ensure(sizeof(DevStatus)));
    CK(cudaEventCreateWithFlags(&h->staging_done, cudaEventDisableTiming));
    h->device_ready = true;
    return DFA_OK;
}

// IdentU8 needs (encoded state) << 8 | byte to be the entry's shared address,
// so |Q| + (table address >> 8) <= 256: measure where dynamic smem starts.
dfa_status probe(dfa_handle *h, uint32_t &u8_limit) {
    CK(h->status.ensure(sizeof(DevStatus)));
    int base = probe_dynamic_smem_base(h->status.as<uint32_t>());
    if (base < 0) return cuda_fail(cudaGetLastError(), "probe_dynamic_smem_base", __LINE__);
    const uint32_t bias = std::max((((uint32_t)base + 255u) & ~255u) >> 8,  // IdentU8
                                   ((uint32_t)base + kPadStride - 1) / kPadStride);  // IdentU8P
    u8_limit = bias >= 256 ? 0 : 256 - bias;
    return DFA_OK;
}

// an event recorded during graph capture must be an external node to be timed later
void record_event(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
}

const char *const kSections[] = {"converge", "lanes", "compose"};
constexpr int kNumSections = 3;

cudaEvent_t prof_event(dfa_handle *h) {
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        h->ev_pool.push_back(e);
    }
    return h->ev_pool[h->ev_used++];
}
void prof_begin(dfa_handle *h, cudaStream_t s, int section) {
    if (!h->profile || h->ev_used + 2 > (1u << 16)) return;
    h->open_event = prof_event(h);
    h->open_section = section;
    if (h->open_event) record_event(h->open_event, s);
}
void prof_end(dfa_handle *h, cudaStream_t s) {
    if (!h->profile || h->open_section < 0 || !h->open_event) return;
    cudaEvent_t b = prof_event(h);
    if (b) {
        record_event(b, s);
        h->recs.push_back({h->open_section, h->open_event, b});
    }
    h->open_section = -1;
}

// Children per composition-tree node: as many as fit a warp's shared-memory
// slice (8 warps per CTA), at most 64.  The rank table is staged as uint8 when
// I_max < 255 and it is small.
uint32_t tree_fanin(const dfa_handle *h, int &rank_smem, int &smem_bytes) {
    const DevTables &T = h->T;
    const uint64_t cap = (uint64_t)h->optin_smem;
    // stage the uint8 rank table in shared memory when it leaves room for F >= 8
    rank_smem = 0;
    if (T.rank8 && (uint64_t)tree_fixed_bytes(T, 1) + (uint64_t)tree_slice_bytes(T, 8) * 8 <= cap) rank_smem = 1;
    const uint64_t fixed = (uint64_t)tree_fixed_bytes(T, rank_smem);
    const uint64_t budget = cap - fixed;
    uint32_t F = h->tree_fanin_cap;
    if (T.rs > 16) F = std::min<uint32_t>(F, h->walk_fanin);  // walk_kernel chains: keep them short
    while (F > 2 && (uint64_t)tree_slice_bytes(T, F) * 8 > budget) F--;
    smem_bytes = (int)(fixed + (uint64_t)tree_slice_bytes(T, F) * 8);
    return F;
}

struct Outputs {
    uint32_t first_dom = 0xFFFFFFFFu; // domain of the first sub-chunk (default: {q0})
    uint16_t *user_row0 = nullptr;   // [imax_user] map of chunk 0 in the user's order (segments)
    uint16_t *chunk0_end = nullptr;  // [1]
    uint16_t *user_maps = nullptr;   // [(P-1) * imax_user]
    uint16_t *starts = nullptr;      // [P]
    uint16_t *final2 = nullptr;      // [2]
    uint16_t *seg_row = nullptr;     // [imax_user] composed map of the whole input over chunk 0's domain
    bool indep = false;              // batch: chunks are independent inputs, no fold
};

int lanes_threads(const dfa_handle *h) {
    if (h->threads_auto) return lanes_max_threads(h->T.mode);
    return std::min(h->threads, lanes_max_threads(h->T.mode));
}

// Execution split of the P reporting chunks (chunk 0 into m0 sub-chunks, the
// others into m): about one sub-chunk per resident thread.  For maps of <= 8
// entries the split is in aligned groups of g = 2^g_log sub-chunks (m0, m
// multiples of g, g | 32 or g = 32) that lanes_kernel composes in the warp.
struct Split {
    uint32_t m0 = 1, m = 1, g_log = kNoWarpGroup;
    int threads = 512;
};

Split plan_split(const dfa_handle *h, uint64_t n, uint32_t P, const uint64_t *hb, bool explicit_bounds) {
    Split sp;
    const int base_threads = lanes_threads(h);
    // one CTA per SM of up to 1024 threads (lanes_max_threads) rather than two of 512 where
    // the table would allow two: same warps, measured +0.5% (Protein) / +0.8% (Keyword)
    const int bps = 1;
    uint64_t target = h->subchunk_target;
    if (target <= 0) {
        target = (uint64_t)h->sms * std::max(1, lanes_occupancy(h->T, base_threads)) * base_threads;
        // converge_kernel costs ~ NS * |I_sigma| while a lanes kernel held to one CTA per SM
        // by a large table is pipe-bound at ~16 warps per SM (Worst, measured: 95k
        // sub-chunks 1499 GB/s, 151k 1388 GB/s): fewer, longer sub-chunks there
        // (measured per layout: Worst/packed9 640 threads per SM 5.89 ms, 768: 5.98; Protein/window_u16
        // 768 threads 1.624 ms, 640: 1.679, 1024: 1.691)
        if (h->convergence && h->T.imax > (uint32_t)kLanes && lanes_occupancy(h->T, 512) < 2)
            target = std::min<uint64_t>(target, (uint64_t)h->sms * (h->T.mode == kPacked9 ? 640 : 768));
        // converge_kernel work per sub-chunk is ~|I_sigma| lanes over the first few hundred
        // bytes whatever the sub-chunk length: keep sub-chunks >= 4 KiB on average so that
        // short inputs (dfa_match_host pieces, segments) are not all convergence
        if (h->convergence && h->T.imax > (uint32_t)kLanes)
            target = std::min<uint64_t>(target, std::max<uint64_t>(1, n / 4096));
    }
    // (explicit partitions need no host bounds: one sub-chunk per chunk)
    const uint64_t len0 = explicit_bounds ? 0 : hb[1] - hb[0];
    uint64_t minlen = len0, avg = len0;
    if (P > 1 && !explicit_bounds) {
        minlen = UINT64_MAX;
        for (uint32_t k = 1; k < P; k++) minlen = std::min(minlen, hb[k + 1] - hb[k]);
        avg = (n - len0) / (P - 1);
    }
    // compose8's last CTA folds <= 1024 CTA maps of <= 1024 chunks: P > 2^20 takes the tree path
    const bool warp_mode = h->T.rs == 8 && h->warp_compose && !h->fold_in_tree && P <= (1u << 20);
    if (explicit_bounds) {
        sp.m0 = sp.m = 1;
        if (warp_mode) sp.g_log = 0;
    } else if (!warp_mode) {
        const uint64_t Ls = std::max<uint64_t>(32, (n + target - 1) / target);
        sp.m0 = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(1, (len0 + Ls / 2) / Ls), std::min<uint64_t>(len0, 1u << 30));
        sp.m = P > 1 ? (uint32_t)std::min<uint64_t>(std::max<uint64_t>(1, (avg + Ls / 2) / Ls), minlen) : 1;
        // rounding to the nearest split can exceed the resident threads, and the excess
        // sub-chunks would run as a second wave (Protein P = 32768: 163,840 sub-chunks for
        // 151,552 threads, 1694 GB/s; 2072 after rounding down)
        const uint64_t slots = (uint64_t)h->sms * bps * std::min(bps >= 2 ? 512 : 1024, lanes_max_threads(h->T.mode));
        while (sp.m > 1 && (uint64_t)sp.m0 + (uint64_t)(P - 1) * sp.m > slots) sp.m--;
        // a sub-chunk stride that is a multiple of 8 KiB puts a warp's 32 streams on the same
        // memory partitions (Protein, 1 MiB chunks in 32 parts: 1.82 ms vs 1.62 ms in 27)
        while (sp.m > 1 && avg / sp.m >= 8192 && (avg / sp.m) % 8192 == 0 && avg % sp.m == 0) sp.m--;
        while (sp.m0 > 1 && (uint64_t)sp.m0 + (uint64_t)(P - 1) * sp.m > slots) sp.m0--;
    } else {
        // sub-chunks of >= 32 bytes; m a multiple of the largest power-of-two group
        // g <= 32 that keeps >= 95% of the estimated split (whole groups per warp)
        auto shape = [](uint64_t est) {
            est = std::max<uint64_t>(est, 1);
            for (uint64_t g = 32; g > 1; g /= 2)
                if (est >= g && (est / g * g) * 100 >= est * DFA_SHAPE_PCT) return (uint32_t)(est / g * g);
            return (uint32_t)est;
        };
        auto group_of = [](uint32_t m) { uint32_t g = 1; while (g < 32 && m % (2 * g) == 0) g *= 2; return g; };
        uint32_t g;
        if (P == 1) {
            sp.m0 = shape(std::min<uint64_t>(target, std::max<uint64_t>(1, len0 / 32)));
            g = group_of(sp.m0);
            sp.m = 1;
        } else {
            const double c = (double)len0 / (double)std::max<uint64_t>(avg, 1);
            const uint64_t est = (uint64_t)((double)target / ((double)(P - 1) + c));
            sp.m = shape(std::min<uint64_t>(est, std::max<uint64_t>(1, minlen / 32)));
            // (a stride that is a multiple of 8 KiB: see below; Keyword 64 KiB chunks in 8: 0.467 vs 0.442 ms)
            if (sp.m > 1 && avg % sp.m == 0 && (avg / sp.m) % 8192 == 0) sp.m = shape(sp.m - 1);
            g = group_of(sp.m);
            uint64_t m0 = (uint64_t)((double)sp.m * c + 0.5);
            m0 = std::max<uint64_t>(g, m0 / g * g);
            while (m0 > len0 && m0 > g) m0 -= g;
            while (len0 < m0 && g > 1) { g /= 2; m0 = std::max<uint64_t>(g, m0 / 2); }
            if (sp.m % g) sp.m = std::max<uint32_t>(g, sp.m / g * g);  // chunk 0 too short: smaller groups
            sp.m0 = (uint32_t)m0;
        }
        uint32_t gl = 0;
        while ((1u << gl) < g) gl++;
        sp.g_log = gl;
    }
    // threads per CTA: spread the sub-chunks evenly over all SMs (one wave when possible)
    const uint64_t NS = (uint64_t)sp.m0 + (uint64_t)(P - 1) * sp.m;
    // small splits (Tiny) keep two CTAs per SM where the table allows: shorter CTAs start sooner
    const int bpt = NS * 2 >= (uint64_t)h->sms * lanes_max_threads(h->T.mode)
                        ? bps : std::max(1, std::min(2, lanes_occupancy(h->T, 512)));
    const int maxt = std::min(bpt >= 2 ? 512 : 1024, lanes_max_threads(h->T.mode));
    uint64_t t = (NS + (uint64_t)h->sms * bpt - 1) / ((uint64_t)h->sms * bpt);
    t = (t + 31) / 32 * 32;
    sp.threads = h->threads_auto ? (int)std::min<uint64_t>(std::max<uint64_t>(t, 128), (uint64_t)maxt) : base_threads;
    return sp;
}

// Core: match `in` under the partition dev_bounds[P+1] (already on the device).
dfa_status run(dfa_handle *h, const uint8_t *in, uint64_t n, uint32_t P, const uint64_t *dev_bounds,
               const Split &sp, cudaStream_t s, const Outputs &o) {
    const uint32_t m0 = sp.m0, m = sp.m;
    DevTables &T = h->T;
    h->stats.input_bytes = 0;
    h->last_stream = s;
    CK(cudaMemsetAsync(h->status.p, 0, sizeof(DevStatus), s));
    unsigned long long *work = nullptr;
    if (h->count_work) {
        CK(h->work.ensure(16));
        if (!h->work_pending) CK(cudaMemsetAsync(h->work.p, 0, 16, s));
        h->work_pending = true;
        h->work_calls++;
        work = h->work.as<unsigned long long>();
    }
    Plan plan{n, P, m0, m, (uint64_t)m0 + (uint64_t)(P - 1) * m, dev_bounds,
              o.first_dom == 0xFFFFFFFFu ? T.start_dom : o.first_dom, (uint64_t)(uintptr_t)in, o.indep ? 1u : 0u,
              work, 0u, 0u, nullptr, plan_magic(m0), plan_magic(m)};
    const uint64_t NS = plan.NS;
    h->stats.input_bytes = n;
    h->stats.num_subchunks = NS;

    // stage A: lock-step convergence of large initial-state sets
    // (link codes of converge_kernel need |Q| <= 0x7F00; larger automata run every lane in
    // lanes_kernel passes)
    const bool stageA = h->convergence && T.imax > (uint32_t)kLanes && T.nq <= 0x7F00u;
    int wpc = 0;
    if (stageA) {
        // as many warps per SM as the table leaves scratch for (the stage is latency- and
        // issue-bound: Worst 16 -> 27 warps), spread over the SMs when NS is small
        for (int w = 32; w >= 1; w--)
            if (converge_smem_bytes(T, w) <= h->optin_smem) { wpc = w; break; }
        const uint64_t per_sm = (NS + h->sms - 1) / h->sms;
        if (wpc) wpc = (int)std::min<uint64_t>((uint64_t)wpc, std::max<uint64_t>(4, per_sm));
    }
    const uint32_t sk = stageA && wpc ? (uint32_t)kLanes : std::max<uint32_t>(kLanes, T.rs);
    CK(h->sfin.ensure(NS * sk * 2));
    CK(h->dom_of.ensure(NS * 2));
    const uint16_t *amap = nullptr, *surv = nullptr;
    const uint8_t *surv_n = nullptr;
    const uint64_t *surv_pos = nullptr;
    int kernels = 0;
    const bool grouped = sp.g_log != kNoWarpGroup;
    // long rows behind the converge stage compose in factored form (fchunk/fwalk/ffold): the
    // converge maps stay coded, and internal sub-chunks may start from the two-symbol sets
    const bool factored = stageA && wpc && !grouped && T.rs > 16 && h->factored;
    plan.keep_amap = factored ? 1u : 0u;
    plan.use_dom2 = factored && h->lookahead2 ? 1u : 0u;
    if (stageA && wpc) {
        CK(h->surv.ensure(NS * kLanes * 2));
        CK(h->surv_n.ensure(NS));
        CK(h->surv_pos.ensure(NS * 8));
        CK(h->amap.ensure(NS * T.rs * 2));
        const int occ = std::max(1, converge_occupancy(T, wpc));
        const uint64_t grid = std::min<uint64_t>((uint64_t)h->sms * occ, (NS + wpc - 1) / wpc);
        prof_begin(h, s, 0);
        CK(launch_converge(T, plan, in, h->surv.as<uint16_t>(), h->surv_n.as<uint8_t>(), h->surv_pos.as<uint64_t>(),
                           h->amap.as<uint16_t>(), (uint32_t)h->max_lanes, wpc, (int)grid, s));
        prof_end(h, s);
        kernels++;
        amap = h->amap.as<uint16_t>();
        surv = h->surv.as<uint16_t>();
        surv_n = h->surv_n.as<uint8_t>();
        surv_pos = h->surv_pos.as<uint64_t>();
    }

    const int threads = sp.threads;
    const int occ = std::max(1, lanes_occupancy(T, threads));
    const uint64_t grid = std::min<uint64_t>((uint64_t)h->sms * occ, (NS + threads - 1) / threads);
    // fused composition tail (one sub-chunk per thread, so CTAs hold contiguous leaves):
    // the lanes kernel composes its own leaves, no leaf_fold / compose8 launches
    const bool fused = grouped && h->fused_tail && !o.indep && !o.seg_row && NS <= grid * (uint64_t)threads && P <= (1u << 20) &&
                       (threads >> sp.g_log) <= 1024;
    Fuse fz{};
    if (fused) {
        fz.on = 1;
        fz.rows = (o.user_maps || o.user_row0 || o.chunk0_end) ? 1u : 0u;
        fz.L0 = m0 >> sp.g_log;
        fz.L = P > 1 ? (m >> sp.g_log) : 1;
        fz.P = P;
        CK(h->lvlA.ensure((uint64_t)P * T.rs * 2));
        CK(h->domA.ensure((uint64_t)P * 2));
        CK(h->part_rows.ensure(((uint64_t)P + grid) * 16));
        CK(h->part_doms.ensure(((uint64_t)P + grid) * 2));
        if (h->chunk_cnt.cap < (uint64_t)P * 4) {
            CK(h->chunk_cnt.ensure((uint64_t)P * 4));
            CK(cudaMemsetAsync(h->chunk_cnt.p, 0, h->chunk_cnt.cap, s));  // then reset by the last arrivers
        }
        CK(h->fold_rows.ensure(grid * 16 + 256));
        CK(h->fold_doms.ensure(grid * 2 + 256));
        if (!h->ticket.p) {
            CK(h->ticket.ensure(256));
            CK(cudaMemsetAsync(h->ticket.p, 0, 256, s));
        }
        fz.rep_rows = h->lvlA.as<uint16_t>();
        fz.rep_doms = h->domA.as<uint16_t>();
        fz.user_rows = o.user_maps;
        fz.user_row0 = o.user_row0;
        fz.e0 = o.chunk0_end;
        fz.part_rows = h->part_rows.as<uint16_t>();
        fz.part_doms = h->part_doms.as<uint16_t>();
        fz.chunk_cnt = h->chunk_cnt.as<uint32_t>();
        fz.cta_rows = h->fold_rows.as<uint16_t>();
        fz.cta_doms = h->fold_doms.as<uint16_t>();
        fz.ticket = h->ticket.as<uint32_t>();
        fz.final2 = o.final2;
        if (o.starts) {
            CK(h->cta_start.ensure(grid * 2 + 256));
            fz.starts = o.starts;
            fz.cta_code = h->cta_start.as<uint16_t>();
        }
    }
    if (grouped) {
        CK(h->leaf_rows.ensure(((NS >> sp.g_log) + 1) * T.rs * 2));
        CK(h->leaf_dom.ensure(((NS >> sp.g_log) + 1) * 2));
    }
    // TMA input staging (run_lanes_tma): one sub-chunk per thread, maps kept in registers, a
    // layout it is built for.  The input as overlapping 64-byte rows at a 32-byte pitch from
    // its 32-byte aligned base; rows that would end past the input are left to the byte loop.
    plan.tmap = nullptr;
    if (h->tma_input && grouped && !fused && !h->count_work && h->max_lanes >= kLanes && NS <= grid * (uint64_t)threads &&
        lanes_tma_available(T, threads, h->optin_smem) && encode_tiled_fn()) {
        const uint64_t addr = (uint64_t)(uintptr_t)in, base = addr & ~31ull, L = addr + n - base;
        const uint64_t rows = L >= 64 ? (L - 64) / 32 + 1 : 0;
        if (rows && rows < (1ull << 32)) {
            if (!h->tmap.p || base != h->tmap_base || rows != h->tmap_rows) {
                const cuuint64_t dims[2] = {64, rows}, strides[1] = {32};
                const cuuint32_t box[2] = {64, 1}, estr[2] = {1, 1};
                const CUresult cr = encode_tiled_fn()(&h->tmap_host, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                                                      reinterpret_cast<void *>((uintptr_t)base), dims, strides, box, estr,
                                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (cr == CUDA_SUCCESS) {
                    CK(h->tmap.ensure(sizeof(CUtensorMap)));
                    g_scratch_gen++;  // a captured graph of another input must not replay against this map
                    CK(cudaMemcpyAsync(h->tmap.p, &h->tmap_host, sizeof(CUtensorMap), cudaMemcpyHostToDevice, s));
                    h->tmap_base = base;
                    h->tmap_rows = rows;
                } else {
                    h->tmap_base = h->tmap_rows = 0;
                }
            }
            if (h->tmap_base == base && h->tmap_rows == rows) plan.tmap = h->tmap.p;
        }
    }
    {
        prof_begin(h, s, 1);
        CK(launch_lanes(T, plan, in, surv, surv_n, surv_pos, h->sfin.as<uint16_t>(), sk, h->dom_of.as<uint16_t>(),
                        h->convergence, const_cast<uint16_t *>(amap), sp.g_log, h->leaf_rows.as<uint16_t>(),
                        h->leaf_dom.as<uint16_t>(), h->status.as<DevStatus>(), (uint32_t)h->max_lanes, threads,
                        (int)grid, s, fz));
        prof_end(h, s);
        kernels++;
    }
    if (fused) {
        if (o.starts) {
            CK(launch_fused_starts(T, plan, fz, in, (uint32_t)(threads >> sp.g_log), sp.g_log, (int)grid, s));
            kernels++;
        }
        h->rep_rows = h->lvlA.as<uint16_t>();
        h->rep_rs = 8;
        h->stats.num_kernels = kernels;
        return DFA_OK;
    }
    // composition: sub-chunk maps -> reporting maps -> final state
    if (grouped) {
        // rank-space leaves (maps of <= 8 entries): leaf_fold passes while the
        // chunks hold more than 64 leaves, then compose8_kernel
        uint32_t L0 = m0 >> sp.g_log, Lm = P > 1 ? (m >> sp.g_log) : 1;
        CK(h->lvlA.ensure((uint64_t)P * T.rs * 2));
        CK(h->domA.ensure((uint64_t)P * 2));
        uint16_t *lrows = h->leaf_rows.as<uint16_t>(), *ldom = h->leaf_dom.as<uint16_t>();
        prof_begin(h, s, 2);
        if (L0 > 64 || Lm > 64) {
            const uint64_t n1 = (uint64_t)(L0 + 31) / 32 + (uint64_t)(P - 1) * ((Lm + 31) / 32) + 1;
            CK(h->leaf_rows2.ensure(n1 * T.rs * 2));
            CK(h->leaf_dom2.ensure(n1 * 2));
            uint16_t *orows = h->leaf_rows2.as<uint16_t>(), *odom = h->leaf_dom2.as<uint16_t>();
            while (L0 > 64 || Lm > 64) {
                CK(launch_leaf_fold(lrows, ldom, L0, Lm, P, orows, odom, h->sms, s));
                kernels++;
                L0 = (L0 + 31) / 32;
                Lm = (Lm + 31) / 32;
                std::swap(lrows, orows);
                std::swap(ldom, odom);
            }
        }
        // chunks per compose8 CTA: 4 per warp, spread over the SMs (one round when
        // P <= 4 * 32 * SMs), at least P / 1024 (the last CTA folds <= 1024 maps)
        uint32_t cpc = std::max<uint32_t>(4, (P + h->sms - 1) / h->sms);
        cpc = (cpc + 3) / 4 * 4;
        if (cpc > 128) cpc = (cpc + 127) / 128 * 128;
        cpc = std::min<uint32_t>(1024, std::max<uint32_t>(cpc, (P + 1023) / 1024));
        const uint32_t g2 = (P + cpc - 1) / cpc;
        CK(h->fold_rows.ensure((uint64_t)g2 * T.rs * 2 + 256));
        CK(h->fold_doms.ensure((uint64_t)g2 * 2 + 256));
        if (o.starts) CK(h->cta_start.ensure((uint64_t)g2 * 2 + 256));
        if (!h->ticket.p) {
            CK(h->ticket.ensure(256));
            CK(cudaMemsetAsync(h->ticket.p, 0, 256, s));
        }
        uint16_t *rep_rows = h->lvlA.as<uint16_t>(), *rep_doms = h->domA.as<uint16_t>();
        h->rep_rows = rep_rows;
        h->rep_rs = 8;
        CK(launch_compose8(T, lrows, ldom, L0, Lm, P, cpc, rep_rows,
                           rep_doms, o.user_maps, o.user_row0, o.chunk0_end, h->fold_rows.as<uint16_t>(),
                           h->fold_doms.as<uint16_t>(), h->ticket.as<uint32_t>(), h->status.as<DevStatus>(), o.final2,
                           h->cta_start.as<uint16_t>(), o.starts, o.seg_row, s));
        prof_end(h, s);
        kernels += o.starts ? 2 : 1;
        h->stats.num_kernels = kernels;
        return DFA_OK;
    }
    Tree tr{};
    bool use_fold_rows = false;
    int tree_smem = 0;
    const uint32_t F = tree_fanin(h, tr.rank_smem, tree_smem);
    tr.F = F;
    {
        uint32_t L = 0;
        uint64_t total = 0;
        struct Sh { uint64_t f, m, S; };
        const uint32_t gl = grouped ? sp.g_log : 0;
        Sh cur{m0 >> gl, P > 1 ? (m >> gl) : 0, P};
        bool overflow = false;
        auto add = [&](Sh prev, uint32_t G) {
            L++;
            if (L > (uint32_t)kMaxLevels) { overflow = true; return Sh{1, 1, 1}; }
            const uint64_t gf = (prev.f + G - 1) / G, gm = prev.S > 1 ? (prev.m + G - 1) / G : 0;
            TreeLevel &lv = tr.lv[L];
            lv.f = (uint32_t)prev.f;
            lv.m = (uint32_t)std::max<uint64_t>(prev.m, 1);
            lv.S = (uint32_t)prev.S;
            lv.G = G;
            lv.gf = (uint32_t)gf;
            lv.gm = (uint32_t)std::max<uint64_t>(gm, 1);
            lv.nodes = (uint32_t)(gf + (prev.S - 1) * gm);
            lv.off = (uint32_t)total;
            total += lv.nodes;
            return Sh{gf, gm, prev.S};
        };
        if (cur.f == 1 && (cur.S == 1 || cur.m == 1)) cur = add(cur, 1);  // leaves are the chunks
        while (!overflow && !(cur.f == 1 && (cur.S == 1 || cur.m == 1))) cur = add(cur, F);
        tr.rep_level = L;
        // short rows: the fold above the reporting chunks is fold_rows_kernel
        // (whole CTAs, pairwise in shared memory); long rows: more tree levels
        use_fold_rows = T.rs <= 16 && P > 1 && !h->fold_in_tree && !o.indep;
        Sh fold{P, 0, 1};
        while (!overflow && !use_fold_rows && !o.indep && fold.f > 1) fold = add(fold, F);
        if (overflow || total >= (1ull << 31) || NS >= (1ull << 31)) return DFA_ERR_INTERNAL;
        tr.nlevels = L;
        tr.root_final = use_fold_rows || o.indep ? 0 : 1;
        tr.lrs = tree_lrs(T);
        CK(h->lvlA.ensure(total * T.rs * 2));
        CK(h->domA.ensure(total * 2));
        if (factored) {
            CK(h->node_nv.ensure(total * 2));
            CK(h->node_fl.ensure(total * 4));
            CK(h->rep_full.ensure((uint64_t)P * T.rs * 2));
            CK(h->clinks.ensure(((uint64_t)P / 8 + 1) * 16));
        }
        // arrival counters: valid across calls with the same tree (multiples of
        // the child counts), zeroed when the tree changes
        std::vector<uint64_t> sig = {total, F, L, (uint64_t)m0, (uint64_t)m, (uint64_t)P, (uint64_t)gl};
        if (sig != h->tree_sig || h->counters.cap < total * 4) {
            g_scratch_gen++;
            CK(h->counters.ensure(total * 4));
            CK(cudaMemsetAsync(h->counters.p, 0, total * 4, s));
            h->tree_sig = sig;
        }
    }
    tr.amap = grouped ? nullptr : amap;
    tr.sfin = grouped ? h->leaf_rows.as<uint16_t>() : h->sfin.as<uint16_t>();
    tr.sk = grouped ? T.rs : sk;
    tr.dom_of = grouped ? h->leaf_dom.as<uint16_t>() : h->dom_of.as<uint16_t>();
    tr.rows = h->lvlA.as<uint16_t>();
    tr.doms = h->domA.as<uint16_t>();
    tr.counters = h->counters.as<uint32_t>();
    tr.user_rows = o.user_maps;
    tr.e0 = o.chunk0_end;
    tr.dev_final = o.final2;
    tr.user_row0 = o.user_row0;
    tr.seg_row = o.seg_row;
    tr.status = h->status.as<DevStatus>();
    if (factored) {
        tr.leaf_nv = surv_n;
        tr.node_nv = h->node_nv.as<uint16_t>();
        tr.node_fl = h->node_fl.as<uint32_t>();
        tr.rep_full = h->rep_full.as<uint16_t>();
    }
    if (T.rs <= 16) {
        const uint64_t warps = tr.lv[1].nodes;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tree_fn(), 256, tree_smem);
        const uint64_t grid = std::min<uint64_t>((warps + 7) / 8, (uint64_t)h->sms * std::max(1, occ));
        prof_begin(h, s, 2);
        CK(launch_tree(T, tr, (int)std::max<uint64_t>(1, grid), tree_smem, s));
        kernels++;
        if (use_fold_rows) {
            const uint32_t lrs = tree_lrs(T);
            const uint64_t budget = (uint64_t)h->optin_smem - 1024 - 64 - fold_rows_fixed_bytes(T);
            // spread the rows over many SMs (single-SM issue rate bounds a lone CTA):
            // about sqrt(P) rows per CTA, the last CTA folds the CTA maps
            const uint32_t cap = (uint32_t)std::min<uint64_t>(budget / ((2ull << lrs) + 2), 8192);
            uint32_t per_cta = 16;
            while ((uint64_t)per_cta * per_cta < P && per_cta < cap) per_cta *= 2;
            per_cta = std::min(per_cta, cap);
            const uint32_t grid = (P + per_cta - 1) / per_cta;
            CK(h->fold_rows.ensure((uint64_t)grid * T.rs * 2 + 256));
            CK(h->fold_doms.ensure((uint64_t)grid * 2 + 256));
            if (!h->ticket.p) {
                CK(h->ticket.ensure(256));
                CK(cudaMemsetAsync(h->ticket.p, 0, 256, s));
            }
            const uint16_t *rep_rows = tr.rows + (uint64_t)tr.lv[tr.rep_level].off * T.rs;
            CK(launch_fold_rows(T, rep_rows, tr.doms + tr.lv[tr.rep_level].off, P, per_cta,
                                h->fold_rows.as<uint16_t>(), h->fold_doms.as<uint16_t>(), h->ticket.as<uint32_t>(),
                                h->status.as<DevStatus>(), o.final2, o.seg_row, s));
            kernels++;
        }
        prof_end(h, s);
    } else {
        // long rows: one entry-parallel launch per level (small fan-in, see tree_fanin)
        prof_begin(h, s, 2);
        // factored: the levels up to the reporting chunks in one launch (a warp per chunk of
        // <= fchunk_cap() leaves), else a launch per level
        const bool chunk_pass = factored && tr.lv[1].S == P && tr.lv[1].f <= fchunk_cap() &&
                                (P == 1 || tr.lv[1].m <= fchunk_cap());
        if (chunk_pass) {
            // (its group links feed ffold_kernel when the reporting level is the one it folds)
            tr.clinks = tr.root_final && P > 1 && P <= ffold_cap() ? h->clinks.as<uint16_t>() : nullptr;
            CK(launch_fchunk(T, tr, h->sms, s));
            kernels++;
        }
        for (uint32_t L = chunk_pass ? tr.rep_level : 1; L <= tr.nlevels; L++) {
            if (!factored) {
                CK(launch_walk(T, tr, L, h->sms, s));
                kernels++;
                continue;
            }
            if (!(chunk_pass && L == tr.rep_level)) {  // (fchunk_kernel wrote the reporting level)
                CK(launch_fwalk(T, tr, L, h->sms, s));
                kernels++;
            }
            if (L == tr.rep_level || (L == tr.nlevels && tr.root_final)) {
                CK(launch_fexpand(T, tr, L, h->sms, s));
                kernels++;
            }
            // the levels above the reporting chunks: one CTA folds them in shared memory
            // once they fit (no launch per level)
            if (L >= tr.rep_level && L < tr.nlevels && tr.root_final && tr.lv[L].nodes <= ffold_cap()) {
                CK(launch_ffold(T, tr, L, s));
                kernels++;
                break;
            }
        }
        prof_end(h, s);
    }
    h->rep_rows = factored ? tr.rep_full : tr.rows + (uint64_t)tr.lv[tr.rep_level].off * T.rs;
    h->rep_rs = T.rs;
    if (o.starts) {
        const uint16_t *rep_rows = h->rep_rows;
        CK(launch_starts(T, plan, rep_rows, rep_rows + T.rs, tr.doms + tr.lv[tr.rep_level].off, o.starts,
                         h->status.as<DevStatus>(), s));
        kernels++;
    }
    h->stats.num_kernels = kernels;
    return DFA_OK;
}

dfa_status check_ready(dfa_handle *h) {
    if (!h) return DFA_ERR_ARG;
    if (!h->device_ready) return DFA_ERR_ARG;
    return DFA_OK;
}

dfa_status stage_bounds(dfa_handle *h, uint64_t n, uint32_t P) {
    if (h->staging_pending) { CK(cudaEventSynchronize(h->staging_done)); h->staging_pending = false; }
    CK(h->h_bounds.ensure((size_t)(P + 1) * 8));
    uint64_t *hb = h->h_bounds.as<uint64_t>();
    for (uint32_t k = 0; k <= P; k++) hb[k] = cform_bound(n, P, h->c_num, h->c_den, k);
    return DFA_OK;
}

dfa_status fetch_status(dfa_handle *h, cudaStream_t s, DevStatus &out) {
    CK(cudaMemcpyAsync(h->h_status.p, h->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out = *h->h_status.as<DevStatus>();
    return DFA_OK;
}

// Replay a captured CUDA graph of `body` when the same call (gkey) repeats.
// First call: eager.  Second identical call: captured on an internal stream
// (the caller's may be the legacy default stream), instantiated, launched on
// the caller's stream.  Later calls: cudaGraphLaunch only.
template <class Body>
dfa_status run_graphed(dfa_handle *h, const std::vector<uint64_t> &gkey, cudaStream_t s, Body body) {
    if (!h->use_graphs || h->count_work) return body(s);  // counters: eager (memset + call count per call)
    if (h->graph_exec && gkey == h->graph_key) {
        CK(cudaGraphLaunch(h->graph_exec, s));
        h->recs = h->graph_recs;
        h->stats.num_kernels = h->graph_kernels;
        h->last_stream = s;
        return DFA_OK;
    }
    if (gkey != h->graph_pending) {
        h->graph_pending = gkey;
        return body(s);
    }
    if (h->graph_exec) { cudaGraphExecDestroy(h->graph_exec); h->graph_exec = nullptr; }
    if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    const uint64_t gen0 = g_scratch_gen.load();
    h->recs.clear();
    h->ev_used = 0;
    CK(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeRelaxed));
    dfa_status st = body(h->cap_stream);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (st != DFA_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture", __LINE__);
    e = cudaGraphInstantiate(&h->graph_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { h->graph_exec = nullptr; return cuda_fail(e, "cudaGraphInstantiate", __LINE__); }
    // scratch reallocated while capturing: the graph would hold stale pointers
    h->graph_key = g_scratch_gen.load() == gen0 ? gkey : std::vector<uint64_t>{};
    // the graph owns the events it records: take them out of the pool
    for (auto &gr : h->graph_recs) { cudaEventDestroy(gr.a); cudaEventDestroy(gr.b); }
    h->graph_recs = h->recs;
    {
        std::vector<cudaEvent_t> keep;
        for (size_t i = 0; i < h->ev_pool.size(); i++) {
            bool owned = false;
            for (auto &gr : h->graph_recs) owned |= (gr.a == h->ev_pool[i] || gr.b == h->ev_pool[i]);
            if (!owned) keep.push_back(h->ev_pool[i]);
        }
        h->ev_pool = keep;
        h->ev_used = 0;
    }
    h->graph_kernels = h->stats.num_kernels;
    CK(cudaGraphLaunch(h->graph_exec, s));
    h->last_stream = s;
    return DFA_OK;
}

} // namespace

extern "C" {

const char *dfa_error_detail(void) { return g_detail; }

const char *dfa_status_string(dfa_status s) {
    switch (s) {
    case DFA_OK: return "ok";
    case DFA_ERR_ARG: return "invalid argument";
    case DFA_ERR_STATES: return "invalid states (|Q| == 0 or > 65000, q0 or a table entry >= |Q|)";
    case DFA_ERR_ALPHABET: return "invalid alphabet size (must be 1..256)";
    case DFA_ERR_CHUNKS: return "invalid chunk count or bounds (some chunk would be empty)";
    case DFA_ERR_SYMBOL: return "input byte outside the alphabet";
    case DFA_ERR_OOM: return "out of memory";
    case DFA_ERR_CUDA: return "CUDA error";
    case DFA_ERR_INTERNAL: return "internal consistency check failed";
    }
    return "unknown status";
}

dfa_status dfa_create_ex(const uint16_t *table, uint32_t num_states, uint32_t alphabet_size, uint16_t q0,
                         const uint8_t *accept_bitmap, uint32_t flags, dfa_handle_t *out) {
    if (!out) return DFA_ERR_ARG;
    std::unique_ptr<dfa_handle> h(new (std::nothrow) dfa_handle());
    if (!h) return DFA_ERR_OOM;
    uint32_t budget = 200 * 1024, rep_budget = 223 * 1024;
    uint32_t u8_limit = 256 - 4;  // dynamic smem starts at shared address 0x400 on sm_100
    if (!(flags & DFA_CREATE_HOST_ONLY)) {
        int dev = 0, optin = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return DFA_ERR_CUDA;
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess && optin > 0) {
            budget = (uint32_t)optin - 24 * 1024;
            rep_budget = (uint32_t)optin - 4 * 1024;  // lanes kernel only: table + bitmaps
        }
        dfa_status ps = probe(h.get(), u8_limit);
        if (ps != DFA_OK) return ps;
    }
    if (flags & ~(uint32_t)(DFA_CREATE_HOST_ONLY | DFA_CREATE_FULL_DOMAIN | DFA_CREATE_TABLE_MODE(0xF)))
        return DFA_ERR_ARG;
    int st = prepare(table, num_states, alphabet_size, q0, accept_bitmap, budget, u8_limit, h->prep,
                     (flags & DFA_CREATE_FULL_DOMAIN) != 0, rep_budget, (int)((flags >> 8) & 0xFu));
    if (st != 0) return (dfa_status)st;
    if (!(flags & DFA_CREATE_HOST_ONLY)) {
        dfa_status ds = upload(h.get());
        if (ds != DFA_OK) { dfa_destroy(h.release()); return ds; }
    }
    *out = h.release();
    return DFA_OK;
}

dfa_status dfa_create(const uint16_t *table, uint32_t num_states, uint32_t alphabet_size, uint16_t q0,
                      const uint8_t *accept_bitmap, dfa_handle_t *out) {
    return dfa_create_ex(table, num_states, alphabet_size, q0, accept_bitmap, 0, out);
}

dfa_status dfa_destroy(dfa_handle_t h) {
    if (!h) return DFA_ERR_ARG;
    if (h->device_ready) {
        if (h->last_stream) cudaStreamSynchronize(h->last_stream);
        for (DevBuf *b : {&h->tables, &h->status, &h->sfin, &h->dom_of, &h->surv, &h->surv_n, &h->surv_pos,
                          &h->amap, &h->lvlA, &h->domA, &h->counters, &h->bounds, &h->input, &h->fold_rows,
                          &h->fold_doms, &h->ticket, &h->leaf_rows, &h->leaf_dom, &h->plan_bounds, &h->cta_start, &h->leaf_rows2, &h->leaf_dom2,
                          &h->part_rows, &h->part_doms, &h->chunk_cnt})
            b->release();
        h->h_status.release();
        h->h_bounds.release();
        if (h->staging_done) cudaEventDestroy(h->staging_done);
        if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
        for (auto &gr : h->graph_recs) { cudaEventDestroy(gr.a); cudaEventDestroy(gr.b); }
        if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
        for (auto &e : h->ev_pool) if (e) cudaEventDestroy(e);
        if (h->copy_stream) { cudaStreamSynchronize(h->copy_stream); cudaStreamDestroy(h->copy_stream); }
        for (auto &e : h->hm_ev) if (e) cudaEventDestroy(e);
        for (DevBuf *b : {&h->hm_rows, &h->hm_bounds, &h->hm_la, &h->hm_final, &h->batch_bounds, &h->batch_kidx,
                          &h->work, &h->node_nv, &h->node_fl, &h->rep_full, &h->clinks, &h->dom2, &h->tmap})
            b->release();
        h->h_hm.release();
        h->h_batch.release();
    }
    delete h;
    return DFA_OK;
}

dfa_status dfa_get_info(dfa_handle_t h, dfa_info *out) {
    if (!h || !out) return DFA_ERR_ARG;
    const Prep &p = h->prep;
    dfa_info i{};
    i.num_states = p.nq_user;
    i.alphabet_size = p.ns;
    i.num_classes = p.nclass_user;
    i.i_max = p.imax_user_stride;
    uint32_t live = p.nq_user - p.num_dead_user;
    uint32_t g = gcd32(p.imax_user, std::max<uint32_t>(live, 1));
    i.gamma_num = p.imax_user / std::max<uint32_t>(g, 1);
    i.gamma_den = std::max<uint32_t>(live, 1) / std::max<uint32_t>(g, 1);
    i.num_dead = p.num_dead_user;
    i.dead_state = p.first_dead_user;
    i.num_absorbing = p.num_absorbing_user;
    i.table_mode = (uint32_t)p.mode;
    i.table_bytes = p.mode == kGlobalU16 ? 0
                  : p.mode == kIdentU8P ? p.nq * kPadStride
                  : (uint32_t)(p.image.size() * 4) << rep_log_of(p.mode);
    i.c_num = h->c_num;
    i.c_den = h->c_den;
    i.device_ready = h->device_ready ? 1 : 0;
    *out = i;
    return DFA_OK;
}

dfa_status dfa_domain(dfa_handle_t h, uint32_t sigma, uint16_t *out_states, uint32_t *out_count) {
    if (!h || !out_count) return DFA_ERR_ARG;
    if (sigma >= h->prep.ns) return DFA_ERR_SYMBOL;
    const auto &d = h->prep.dom_user[h->prep.byte_class[sigma]];
    if (out_states) std::copy(d.begin(), d.end(), out_states);
    *out_count = (uint32_t)d.size();
    return DFA_OK;
}

dfa_status dfa_set_chunk_ratio(dfa_handle_t h, uint32_t c_num, uint32_t c_den) {
    if (!h || c_num == 0 || c_den == 0 || c_num > (1u << 20) || c_den > (1u << 20)) return DFA_ERR_ARG;
    uint32_t g = gcd32(c_num, c_den);
    h->c_num = c_num / g;
    h->c_den = c_den / g;
    return DFA_OK;
}

dfa_status dfa_plan_bounds(uint64_t n, uint32_t P, uint32_t c_num, uint32_t c_den, uint64_t *host_bounds) {
    if (!host_bounds || P == 0 || c_num == 0 || c_den == 0) return DFA_ERR_ARG;
    // every chunk non-empty iff n >= c + P - 1, i.e. n*b >= a + b(P-1)
    if ((unsigned __int128)n * c_den < (unsigned __int128)c_num + (unsigned __int128)c_den * (P - 1))
        return DFA_ERR_CHUNKS;
    for (uint32_t k = 0; k <= P; k++) host_bounds[k] = cform_bound(n, P, c_num, c_den, k);
    return DFA_OK;
}

dfa_status dfa_match(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, void *stream, uint16_t *final_state,
                     int *accept) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    if (!final_state || !accept || (len && !dev_input)) return DFA_ERR_ARG;
    if (len == 0) {
        *final_state = h->prep.q0;
        *accept = h->prep.accepting[h->prep.q0];
        return DFA_OK;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (h->staging_pending) { CK(cudaEventSynchronize(h->staging_done)); h->staging_pending = false; }
    CK(h->h_bounds.ensure(16));
    CK(h->bounds.ensure(16));
    uint64_t *hb = h->h_bounds.as<uint64_t>();
    hb[0] = 0;
    hb[1] = len;
    CK(cudaMemcpyAsync(h->bounds.p, hb, 16, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(h->staging_done, s));
    h->staging_pending = true;
    const Split sp = plan_split(h, len, 1, hb, false);
    Outputs o;
    st = run(h, dev_input, len, 1, h->bounds.as<uint64_t>(), sp, s, o);
    if (st != DFA_OK) return st;
    DevStatus ds{};
    st = fetch_status(h, s, ds);
    if (st != DFA_OK) return st;
    if (ds.err) return (dfa_status)ds.err;
    *final_state = (uint16_t)ds.final_state;
    *accept = (int)ds.accept;
    return DFA_OK;
}

dfa_status dfa_match_host(dfa_handle_t h, const uint8_t *host_input, uint64_t len, void *stream,
                          uint16_t *final_state, int *accept) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    if (!final_state || !accept || (len && !host_input)) return DFA_ERR_ARG;
    if (len == 0) return dfa_match(h, nullptr, 0, stream, final_state, accept);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    CK(h->input.ensure(len));
    const uint64_t piece = h->host_piece;
    const uint32_t G = (uint32_t)((len + piece - 1) / piece);
    if (G == 1) {
        h->stats.host_bytes = len;
        CK(cudaMemcpyAsync(h->input.p, host_input, len, cudaMemcpyHostToDevice, s));
        return dfa_match(h, h->input.as<uint8_t>(), len, stream, final_state, accept);
    }
    // Pieces g = 0..G-1: piece g is copied on copy_stream while piece g-1 is
    // matched on s as a segment map over I_sigma of the byte before it
    // (dfa_segment_map), and the rows so far are folded (Eq.SeqReduction) into
    // the running state, read back per piece.  Early exit: once a finished
    // piece leaves the run in a state that absorbs every byte, the remaining
    // pieces cannot change the result and are neither copied nor matched.
    if (h->staging_pending) { CK(cudaEventSynchronize(h->staging_done)); h->staging_pending = false; }
    if (!h->copy_stream) CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    while (h->hm_ev.size() < 2 * (size_t)G + 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->hm_ev.push_back(e);
    }
    const uint32_t imu = h->T.imax_user;
    CK(h->hm_rows.ensure((size_t)G * imu * 2));
    CK(h->hm_bounds.ensure((size_t)G * 16));
    CK(h->hm_la.ensure(G));
    CK(h->hm_final.ensure((size_t)G * 4));
    const size_t o_la = (size_t)G * 16, o_st = o_la + ((G + 15) & ~15u), o_fin = o_st + (size_t)G * sizeof(DevStatus);
    CK(h->h_hm.ensure(o_fin + (size_t)G * 4));
    uint8_t *hp = h->h_hm.as<uint8_t>();
    // the pinned staging of a previous call may still be in flight
    CK(cudaStreamSynchronize(s));
    uint64_t *hb = reinterpret_cast<uint64_t *>(hp);
    uint8_t *hla = hp + o_la;
    DevStatus *hst = reinterpret_cast<DevStatus *>(hp + o_st);
    uint16_t *hfin = reinterpret_cast<uint16_t *>(hp + o_fin);
    for (uint32_t g = 0; g < G; g++) {
        const uint64_t off = (uint64_t)g * piece, sz = std::min<uint64_t>(piece, len - off);
        hb[2 * g] = 0;
        hb[2 * g + 1] = sz;
        hla[g] = g ? host_input[off - 1] : 0;
        if (g && hla[g] >= h->prep.ns) return DFA_ERR_SYMBOL;
    }
    CK(cudaMemcpyAsync(h->hm_bounds.p, hb, (size_t)G * 16, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(h->hm_la.p, hla, G, cudaMemcpyHostToDevice, s));
    // earlier work on s may still read h->input: the copies start after it
    CK(cudaEventRecord(h->hm_ev[2 * G], s));
    CK(cudaStreamWaitEvent(h->copy_stream, h->hm_ev[2 * G], 0));
    uint16_t *rows = h->hm_rows.as<uint16_t>();
    uint32_t issued = 0, checked = 0;
    int exit_piece = -1;
    uint64_t copied = 0;
    for (uint32_t g = 0; g < G; g++) {
        if (h->early_exit && g >= 2) {
            // at most 3 pieces in flight (copy of g overlaps the match of g-1, g-2), so
            // that a finished piece's running state is seen while there is input left
            if (g >= 3) CK(cudaEventSynchronize(h->hm_ev[2 * (g - 3) + 1]));
            // pieces finish in order on s: look at the newly finished ones
            while (checked + 1 < g && cudaEventQuery(h->hm_ev[2 * checked + 1]) == cudaSuccess) {
                const uint32_t q = hfin[2 * checked];
                if (q < h->prep.nq && h->prep.absorbing[q]) { exit_piece = (int)checked; break; }
                checked++;
            }
            if (exit_piece >= 0) break;
        }
        const uint64_t off = (uint64_t)g * piece, sz = std::min<uint64_t>(piece, len - off);
        CK(cudaMemcpyAsync(h->input.as<uint8_t>() + off, host_input + off, sz, cudaMemcpyHostToDevice,
                           h->copy_stream));
        copied += sz;
        CK(cudaEventRecord(h->hm_ev[2 * g], h->copy_stream));
        CK(cudaStreamWaitEvent(s, h->hm_ev[2 * g], 0));
        const uint64_t hb2[2] = {0, sz};
        const Split sp = plan_split(h, sz, 1, hb2, false);
        Outputs o;
        o.first_dom = g ? h->prep.byte_class[hla[g]] : h->T.start_dom;
        o.user_row0 = rows + (size_t)g * imu;
        st = run(h, h->input.as<uint8_t>() + off, sz, 1, h->hm_bounds.as<uint64_t>() + 2 * g, sp, s, o);
        if (st != DFA_OK) return st;
        CK(launch_fold_segments(h->T, rows, h->hm_la.as<uint8_t>(), g + 1, h->status.as<DevStatus>(),
                                h->hm_final.as<uint16_t>() + 2 * g, s));
        CK(cudaMemcpyAsync(hst + g, h->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hfin + 2 * g, h->hm_final.as<uint16_t>() + 2 * g, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(h->hm_ev[2 * g + 1], s));
        issued = g + 1;
    }
    CK(cudaStreamSynchronize(s));
    h->last_stream = s;
    h->stats.host_bytes = copied;
    const uint32_t last = exit_piece >= 0 ? (uint32_t)exit_piece : issued - 1;
    uint32_t err = 0;
    for (uint32_t g = 0; g <= last; g++) err = std::max(err, hst[g].err);
    if (err) return (dfa_status)err;
    *final_state = hfin[2 * last];
    *accept = (int)hfin[2 * last + 1];
    if (*final_state == h->prep.poison) return DFA_ERR_SYMBOL;
    return DFA_OK;
}

}  // extern "C"

namespace {
// dfa_chunk_maps and dfa_segment_chunk_maps: lookahead < 0 -> the input starts the string
// (chunk 0 from {q0}, chunk0_out = e0 [1]); lookahead = sigma -> the input is a segment that
// follows a byte sigma (chunk 0 from I_sigma, chunk0_out = its row [i_max]); seg_row (optional)
// = the composed map of the whole input over chunk 0's domain.  dev_bounds may be null.
dfa_status chunk_maps_impl(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, uint32_t P, int32_t lookahead,
                           void *stream, uint64_t *dev_bounds, uint16_t *chunk0_out, uint16_t *dev_maps,
                           uint16_t *dev_chunk_start, uint16_t *dev_final, uint16_t *seg_row) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    if (P == 0) return DFA_ERR_CHUNKS;
    if (!dev_input || !chunk0_out || (P > 1 && !dev_maps)) return DFA_ERR_ARG;
    if (lookahead < -1 || lookahead > 255) return DFA_ERR_ARG;
    if (lookahead >= (int32_t)h->prep.ns) return DFA_ERR_SYMBOL;
    if ((unsigned __int128)len * h->c_den < (unsigned __int128)h->c_num + (unsigned __int128)h->c_den * (P - 1))
        return DFA_ERR_CHUNKS;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // the partition and its execution split depend on (n, P, c, options) only:
    // computed once, kept on the device, copied device-to-device per call
    // (every input plan_split reads besides the device and the table layout, fixed per handle)
    const std::vector<uint64_t> key = {len, P, h->c_num, h->c_den, (uint64_t)h->subchunk_target,
                                       (uint64_t)h->threads, (uint64_t)h->threads_auto, (uint64_t)h->warp_compose,
                                       (uint64_t)h->convergence, (uint64_t)h->fold_in_tree};
    if (key != h->plan_key) {
        st = stage_bounds(h, len, P);
        if (st != DFA_OK) return st;
        const uint64_t *hb = h->h_bounds.as<uint64_t>();
        CK(h->plan_bounds.ensure((size_t)(P + 1) * 8));
        CK(cudaMemcpyAsync(h->plan_bounds.p, hb, (size_t)(P + 1) * 8, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(h->staging_done, s));
        h->staging_pending = true;
        const Split sp0 = plan_split(h, len, P, hb, false);
        h->plan_split_c = {sp0.m0, sp0.m, sp0.g_log, sp0.threads};
        h->plan_key = key;
    }
    Split sp;
    sp.m0 = h->plan_split_c.m0;
    sp.m = h->plan_split_c.m;
    sp.g_log = h->plan_split_c.g_log;
    sp.threads = h->plan_split_c.threads;
    Outputs o;
    if (lookahead < 0) o.chunk0_end = chunk0_out;
    else {
        o.first_dom = h->prep.byte_class[lookahead];
        o.user_row0 = chunk0_out;
    }
    o.user_maps = P > 1 ? dev_maps : nullptr;
    o.starts = dev_chunk_start;
    o.final2 = dev_final;
    o.seg_row = seg_row;
    auto body = [&](cudaStream_t cs) -> dfa_status {
        if (dev_bounds)
            CK(cudaMemcpyAsync(dev_bounds, h->plan_bounds.p, (size_t)(P + 1) * 8, cudaMemcpyDeviceToDevice, cs));
        return run(h, dev_input, len, P, h->plan_bounds.as<uint64_t>(), sp, cs, o);
    };
    // repeated identical calls replay a CUDA graph of the whole call (no launch gaps)
    std::vector<uint64_t> gkey = key;
    for (uint64_t v : {(uint64_t)(uintptr_t)dev_input, (uint64_t)(uintptr_t)dev_bounds,
                       (uint64_t)(uintptr_t)chunk0_out, (uint64_t)(uintptr_t)dev_maps,
                       (uint64_t)(uintptr_t)dev_chunk_start, (uint64_t)(uintptr_t)dev_final,
                       (uint64_t)(uintptr_t)seg_row, (uint64_t)(int64_t)lookahead, (uint64_t)h->profile,
                       (uint64_t)h->convergence, (uint64_t)h->tree_fanin_cap, (uint64_t)h->fold_in_tree,
                       (uint64_t)h->max_lanes, (uint64_t)h->warp_compose, (uint64_t)h->subchunk_target,
                       (uint64_t)h->threads, (uint64_t)h->T.has_sticky, (uint64_t)h->count_work, (uint64_t)h->fused_tail,
                       (uint64_t)h->factored, (uint64_t)h->lookahead2, (uint64_t)h->tma_input,
                       (uint64_t)g_scratch_gen.load()})
        gkey.push_back(v);
    return run_graphed(h, gkey, s, body);
}
}  // namespace

extern "C" {

dfa_status dfa_chunk_maps(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, uint32_t num_chunks, void *stream,
                          uint64_t *dev_bounds, uint16_t *dev_chunk0_end, uint16_t *dev_maps,
                          uint16_t *dev_chunk_start, uint16_t *dev_final) {
    if (h && !dev_bounds) return DFA_ERR_ARG;
    return chunk_maps_impl(h, dev_input, len, num_chunks, -1, stream, dev_bounds, dev_chunk0_end, dev_maps,
                           dev_chunk_start, dev_final, nullptr);
}

dfa_status dfa_segment_chunk_maps(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, uint32_t num_chunks,
                                  int32_t lookahead, void *stream, uint64_t *dev_bounds, uint16_t *dev_chunk0_row,
                                  uint16_t *dev_maps, uint16_t *dev_segment_row) {
    if (h && !dev_segment_row) return DFA_ERR_ARG;
    return chunk_maps_impl(h, dev_input, len, num_chunks, lookahead, stream, dev_bounds, dev_chunk0_row, dev_maps,
                           nullptr, nullptr, dev_segment_row);
}

dfa_status dfa_chunk_maps_at(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, uint32_t num_chunks,
                             const uint64_t *dev_bounds_in, void *stream, uint16_t *dev_chunk0_end,
                             uint16_t *dev_maps, uint16_t *dev_chunk_start, uint16_t *dev_final) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    const uint32_t P = num_chunks;
    if (P == 0 || len < P) return DFA_ERR_CHUNKS;
    if (!dev_input || !dev_bounds_in || !dev_chunk0_end || (P > 1 && !dev_maps)) return DFA_ERR_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    std::vector<uint64_t> hb(P + 1);
    CK(cudaMemcpyAsync(hb.data(), dev_bounds_in, (size_t)(P + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hb[0] != 0 || hb[P] != len) return DFA_ERR_CHUNKS;
    for (uint32_t k = 0; k < P; k++)
        if (hb[k + 1] <= hb[k]) return DFA_ERR_CHUNKS;
    Outputs o;
    o.chunk0_end = dev_chunk0_end;
    o.user_maps = P > 1 ? dev_maps : nullptr;
    o.starts = dev_chunk_start;
    o.final2 = dev_final;
    const Split sp = plan_split(h, len, P, hb.data(), true);
    return run(h, dev_input, len, P, dev_bounds_in, sp, s, o);
}

dfa_status dfa_match_batch(dfa_handle_t h, const uint8_t *dev_data, uint64_t data_len, const uint64_t *dev_offsets,
                           uint32_t count, void *stream, uint16_t *dev_final, uint8_t *dev_accept) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    if (count == 0) return DFA_OK;
    if (!dev_offsets || !dev_final || !dev_accept || (data_len && !dev_data)) return DFA_ERR_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    h->last_stream = s;
    const uint32_t P = count;
    Outputs o;
    o.indep = true;
    if (count >= 4096) {
        // many inputs: the batch is the parallelism -- one sub-chunk per input, the
        // caller's offsets are the partition as they are (empty inputs included), no
        // host round trip; the kernels clamp offsets to data_len and flag bad ones
        const Split sp = plan_split(h, data_len, P, nullptr, true);
        st = run(h, dev_data, data_len, P, dev_offsets, sp, s, o);
        if (st != DFA_OK) return st;
        CK(launch_batch_out(h->T, h->rep_rows, h->rep_rs, nullptr, dev_offsets, data_len, count, dev_final,
                            dev_accept, h->status.as<DevStatus>(), s));
        h->stats.num_kernels++;
        return DFA_OK;
    }
    // few inputs: read the offsets, drop empty inputs, split each input for parallelism
    if (h->staging_pending) { CK(cudaEventSynchronize(h->staging_done)); h->staging_pending = false; }
    CK(h->h_batch.ensure((size_t)(count + 1) * 8 * 2 + (size_t)count * 4 + 64));
    uint64_t *ho = h->h_batch.as<uint64_t>();
    uint64_t *hb = ho + count + 1;
    int32_t *hk = reinterpret_cast<int32_t *>(hb + count + 1);
    CK(cudaMemcpyAsync(ho, dev_offsets, (size_t)(count + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (uint32_t j = 0; j < count; j++)
        if (ho[j + 1] < ho[j]) return DFA_ERR_ARG;
    if (ho[count] > data_len) return DFA_ERR_ARG;
    const uint64_t base = ho[0], n = ho[count] - base;
    uint32_t Pn = 0;
    hb[0] = 0;
    for (uint32_t j = 0; j < count; j++) {
        if (ho[j + 1] > ho[j]) {
            hk[j] = (int32_t)Pn++;
            hb[Pn] = ho[j + 1] - base;
        } else {
            hk[j] = -1;
        }
    }
    CK(h->batch_kidx.ensure((size_t)count * 4));
    CK(cudaMemcpyAsync(h->batch_kidx.p, hk, (size_t)count * 4, cudaMemcpyHostToDevice, s));
    if (Pn == 0) {
        CK(cudaMemsetAsync(h->status.p, 0, sizeof(DevStatus), s));
        CK(launch_batch_out(h->T, nullptr, 8, h->batch_kidx.as<int32_t>(), nullptr, 0, count, dev_final,
                            dev_accept, h->status.as<DevStatus>(), s));
    } else {
        CK(h->batch_bounds.ensure((size_t)(Pn + 1) * 8));
        CK(cudaMemcpyAsync(h->batch_bounds.p, hb, (size_t)(Pn + 1) * 8, cudaMemcpyHostToDevice, s));
        const Split sp = plan_split(h, n, Pn, hb, false);
        st = run(h, dev_data + base, n, Pn, h->batch_bounds.as<uint64_t>(), sp, s, o);
        if (st != DFA_OK) return st;
        CK(launch_batch_out(h->T, h->rep_rows, h->rep_rs, h->batch_kidx.as<int32_t>(), nullptr, 0, count,
                            dev_final, dev_accept, h->status.as<DevStatus>(), s));
        h->stats.num_kernels++;
    }
    // the pinned staging must outlive the async copies above
    CK(cudaEventRecord(h->staging_done, s));
    h->staging_pending = true;
    return DFA_OK;
}

dfa_status dfa_lookahead_maps(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, uint32_t num_chunks,
                              const uint64_t *dev_bounds, const uint16_t *dev_maps, uint32_t r, void *stream,
                              uint16_t *dev_domains, uint16_t *dev_domain_sizes, uint16_t *dev_maps_r) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    const uint32_t P = num_chunks;
    if (P == 0 || len < P) return DFA_ERR_CHUNKS;
    if (r < 1 || r > 16) return DFA_ERR_ARG;
    if (P == 1) return DFA_OK;
    if (!dev_input || !dev_bounds || !dev_maps || !dev_domains || !dev_domain_sizes || !dev_maps_r)
        return DFA_ERR_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    h->last_stream = s;
    CK(cudaMemsetAsync(h->status.p, 0, sizeof(DevStatus), s));
    CK(launch_lookahead(h->T, dev_input, dev_bounds, P, r, dev_maps, dev_domains, dev_domain_sizes, dev_maps_r,
                        h->status.as<DevStatus>(), h->sms, s));
    return DFA_OK;
}

dfa_status dfa_segment_map(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, int32_t lookahead, void *stream,
                           uint16_t *dev_row) {
    // one chunk: its row is the segment map (device-resident plan, graph replay when repeated)
    if (!dev_input || !dev_row || len == 0) return h ? DFA_ERR_ARG : DFA_ERR_ARG;
    return chunk_maps_impl(h, dev_input, len, 1, lookahead, stream, nullptr, dev_row, nullptr, nullptr, nullptr,
                           dev_row);
}

dfa_status dfa_fold_segments(dfa_handle_t h, const uint16_t *dev_rows, const uint8_t *dev_lookahead, uint32_t G,
                             void *stream, uint16_t *dev_final) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    if (!dev_rows || !dev_lookahead || G == 0) return DFA_ERR_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    h->last_stream = s;
    CK(cudaMemsetAsync(h->status.p, 0, sizeof(DevStatus), s));
    CK(launch_fold_segments(h->T, dev_rows, dev_lookahead, G, h->status.as<DevStatus>(), dev_final, s));
    return DFA_OK;
}

dfa_status dfa_gather_ceiling(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, void *stream,
                              uint16_t *dev_out, uint64_t *out_per_thread, uint32_t *out_threads) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    if (!out_per_thread || !out_threads) return DFA_ERR_ARG;
    // the step alone has one dependent chain per thread: it wants every warp slot (1024
    // threads per CTA), whatever CTA size the lanes kernel picks for its own trade-offs
    const int threads = 1024;
    const int grid = h->sms * std::max(1, ceiling_occupancy(h->T, threads));
    const uint64_t T = (uint64_t)grid * threads;
    const uint64_t per = (len / T) & ~31ull;
    *out_threads = (uint32_t)T;
    *out_per_thread = per;
    if (!dev_out) return DFA_OK;  // query
    if (!dev_input || per == 0 || (reinterpret_cast<uintptr_t>(dev_input) & 31u)) return DFA_ERR_ARG;
    CK(launch_ceiling(h->T, dev_input, per, dev_out, threads, grid, reinterpret_cast<cudaStream_t>(stream)));
    return DFA_OK;
}

dfa_status dfa_get_last_device_error(dfa_handle_t h) {
    dfa_status st = check_ready(h);
    if (st != DFA_OK) return st;
    DevStatus ds{};
    st = fetch_status(h, h->last_stream, ds);
    if (st != DFA_OK) return st;
    return (dfa_status)ds.err;
}

dfa_status dfa_set_option(dfa_handle_t h, uint32_t key, int64_t value) {
    if (!h) return DFA_ERR_ARG;
    switch (key) {
    case DFA_OPT_SUBCHUNK_TARGET: if (value < 0) return DFA_ERR_ARG; h->subchunk_target = value; return DFA_OK;
    case DFA_OPT_HOST_PIECE:
        if (value < (1 << 20)) return DFA_ERR_ARG;
        h->host_piece = (uint64_t)value;
        return DFA_OK;
    case DFA_OPT_EARLY_EXIT: h->early_exit = value ? 1 : 0; return DFA_OK;
    case DFA_OPT_MAX_LANES:
        if (value < 1 || value > kLanes) return DFA_ERR_ARG;
        h->max_lanes = (int)value;
        return DFA_OK;
    case DFA_OPT_CONVERGENCE: h->convergence = value ? 1 : 0; return DFA_OK;
    case DFA_OPT_PROFILE: h->profile = value ? 1 : 0; return DFA_OK;
    case DFA_OPT_TREE_FANIN:
        if (value < 2 || value > 64) return DFA_ERR_ARG;
        h->tree_fanin_cap = (uint32_t)value;
        return DFA_OK;
    case DFA_OPT_GRAPHS:
        h->use_graphs = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_WARP_COMPOSE:
        h->warp_compose = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_FOLD_IN_TREE:
        h->fold_in_tree = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_STICKY_PARKING:
        h->sticky_parking = value ? 1 : 0;
        h->T.has_sticky = h->sticky_avail && h->sticky_parking;
        return DFA_OK;
    case DFA_OPT_COUNT_WORK:
        h->count_work = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_FUSED_TAIL:
        h->fused_tail = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_FACTORED:
        h->factored = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_LOOKAHEAD2:
        h->lookahead2 = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_TMA_INPUT:
        h->tma_input = value ? 1 : 0;
        return DFA_OK;
    case DFA_OPT_THREADS_PER_CTA:
        h->threads_auto = value == 0;
        if (value == 0) value = 512;
        if (value < 32 || value > 1024 || value % 32) return DFA_ERR_ARG;
        h->threads = (int)value;
        return DFA_OK;
    }
    return DFA_ERR_ARG;
}

dfa_status dfa_get_stats(dfa_handle_t h, dfa_stats *out) {
    if (!h || !out) return DFA_ERR_ARG;
    dfa_stats s = h->stats;
    for (int i = 0; i < 8; i++) { s.kernel_ms[i] = 0; s.kernel_name[i][0] = 0; }
    s.profiled = 0;
    if (h->device_ready && !h->recs.empty()) {
        CK(cudaEventSynchronize(h->recs.back().b));
        uint32_t calls = 0;
        for (const auto &r : h->recs) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, r.a, r.b));
            s.kernel_ms[r.section] += ms;
            if (r.section == 1) calls++;
        }
        for (int i = 0; i < kNumSections; i++) std::snprintf(s.kernel_name[i], 32, "%s", kSections[i]);
        s.profiled = calls;
        h->recs.clear();
        h->ev_used = 0;
    }
    s.work_lookups[0] = s.work_lookups[1] = 0;
    s.work_calls = 0;
    if (h->device_ready && h->work_pending) {
        unsigned long long w[2] = {0, 0};
        if (h->last_stream) CK(cudaStreamSynchronize(h->last_stream));
        CK(cudaMemcpy(w, h->work.p, 16, cudaMemcpyDeviceToHost));
        s.work_lookups[0] = w[0];
        s.work_lookups[1] = w[1];
        s.work_calls = h->work_calls;
        h->work_pending = false;
        h->work_calls = 0;
    }
    *out = s;
    return DFA_OK;
}

} // extern "C"
