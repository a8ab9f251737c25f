// prep.cpp -- host preprocessing (see prep.h).
#include "prep.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>

namespace dfa {

namespace {
enum { ST_OK = 0, ST_ARG = 1, ST_STATES = 2, ST_ALPHABET = 3 };

inline bool bit(const uint8_t *bm, uint32_t q) { return (bm[q >> 3] >> (q & 7)) & 1; }

// Smallest aligned byte window [base, base + W) (W = 4..128) holding every
// byte outside the largest column class.  Returns W (0 if none).
uint32_t find_window(const Prep &p, uint32_t &base, uint32_t &def_class) {
    std::vector<uint32_t> count(p.nclass, 0);
    for (int b = 0; b < 256; b++) count[p.byte_class[b]]++;
    def_class = uint32_t(std::max_element(count.begin(), count.end()) - count.begin());
    int lo = 256, hi = -1;
    for (int b = 0; b < 256; b++)
        if (p.byte_class[b] != def_class) { lo = std::min(lo, b); hi = std::max(hi, b); }
    if (hi < 0) { base = 0; return 4; }
    for (uint32_t W = 4; W <= 128; W *= 2) {
        uint32_t bs = uint32_t(lo) & ~(W - 1);
        if (uint32_t(hi) < bs + W) { base = bs; return W; }
    }
    return 0;
}
} // namespace

uint64_t cform_bound(uint64_t n, uint32_t P, uint64_t c_num, uint64_t c_den, uint32_t k) {
    if (k == 0) return 0;
    if (k >= P) return n;
    // b_k = floor(n * (a + b(k-1)) / (a + b(P-1))), c = a/b
    unsigned __int128 num = (unsigned __int128)n * (c_num + c_den * (uint64_t)(k - 1));
    unsigned __int128 den = (unsigned __int128)c_num + (unsigned __int128)c_den * (P - 1);
    return (uint64_t)(num / den);
}

int prepare(const uint16_t *table, uint32_t nq, uint32_t ns, uint16_t q0,
            const uint8_t *accept_bitmap, uint32_t smem_budget, uint32_t u8_state_limit, Prep &p,
            bool full_domain, uint32_t rep_budget, int forced_mode) {
    if (!table || !accept_bitmap) return ST_ARG;
    if (ns == 0 || ns > 256) return ST_ALPHABET;
    if (nq == 0 || nq > kMaxStates || q0 >= nq) return ST_STATES;
    for (uint64_t i = 0; i < (uint64_t)nq * ns; i++)
        if (table[i] >= nq) return ST_STATES;

    p = Prep();
    p.nq_user = nq;
    p.ns = ns;
    p.q0 = q0;
    const bool need_poison = ns < 256;
    p.nq = nq + (need_poison ? 1 : 0);
    if (p.nq > kMaxStates) return ST_STATES;
    p.poison = need_poison ? uint16_t(nq) : kNone;

    // internal byte-indexed table
    p.full.assign((size_t)p.nq * 256, 0);
    for (uint32_t q = 0; q < p.nq; q++)
        for (uint32_t b = 0; b < 256; b++) {
            uint16_t t;
            if (q < nq && b < ns) t = table[(size_t)q * ns + b];
            else t = p.poison;  // bytes >= |Sigma| and the poison row
            p.full[(size_t)q * 256 + b] = t;
        }
    p.accepting.assign(p.nq, 0);
    for (uint32_t q = 0; q < nq; q++) p.accepting[q] = bit(accept_bitmap, q);

    // absorbing states and error states Z (reading R1)
    p.absorbing.assign(p.nq, 0);
    p.dead.assign(p.nq, 0);
    for (uint32_t q = 0; q < p.nq; q++) {
        bool ab = true;
        for (uint32_t b = 0; b < 256 && ab; b++) ab = p.full[(size_t)q * 256 + b] == q;
        p.absorbing[q] = ab;
        p.dead[q] = ab && !p.accepting[q];
    }
    // user-visible error states: absorbing over the user alphabet, not accepting
    p.dead_user.assign(p.nq, 0);
    for (uint32_t q = 0; q < nq; q++) {
        bool ab = true;
        for (uint32_t b = 0; b < ns && ab; b++) ab = table[(size_t)q * ns + b] == q;
        if (ab) p.num_absorbing_user++;
        if (ab && !p.accepting[q]) {
            p.dead_user[q] = 1;
            p.num_dead_user++;
            if (p.first_dead_user == kNone) p.first_dead_user = uint16_t(q);
        }
    }
    if (need_poison) p.dead_user[p.poison] = 1;

    // column classes over all 256 bytes of the internal table
    p.byte_class.assign(256, 0);
    {
        std::map<std::vector<uint16_t>, uint32_t> ids;
        std::vector<uint16_t> col(p.nq);
        for (uint32_t b = 0; b < 256; b++) {
            for (uint32_t q = 0; q < p.nq; q++) col[q] = p.full[(size_t)q * 256 + b];
            auto it = ids.find(col);
            if (it == ids.end()) {
                uint32_t id = uint32_t(ids.size());
                ids.emplace(col, id);
                p.class_rep.push_back(uint16_t(b));
                p.byte_class[b] = uint8_t(id);
            } else {
                p.byte_class[b] = uint8_t(it->second);
            }
        }
        p.nclass = uint32_t(ids.size());
    }
    {
        std::vector<uint8_t> valid(p.nclass, 0);
        for (uint32_t b = 0; b < ns; b++) valid[p.byte_class[b]] = 1;
        for (uint32_t c = 0; c < p.nclass; c++) p.nclass_user += valid[c];
    }

    // I_sigma per class, then the {q0} domain of the first sub-chunk
    p.start_dom = p.nclass;
    p.dom.assign(p.nclass + 1, {});
    p.dom_user.assign(p.nclass, {});
    p.xlat.assign(p.nclass, {});
    std::vector<uint8_t> mark(p.nq);
    // Alg.2 ablation (full_domain): every sub-chunk is matched from all states
    // Q \ Z; the API rows stay over I_sigma, read out of the
    // full map through xlat.
    std::vector<uint16_t> full_idx(p.nq, kNone), live;
    for (uint32_t q = 0; q < p.nq; q++)
        if (!p.dead[q]) { full_idx[q] = uint16_t(live.size()); live.push_back(uint16_t(q)); }
    p.full_domain = full_domain;
    for (uint32_t c = 0; c < p.nclass; c++) {
        std::fill(mark.begin(), mark.end(), 0);
        uint32_t b = p.class_rep[c];
        for (uint32_t q = 0; q < p.nq; q++) mark[p.full[(size_t)q * 256 + b]] = 1;
        if (full_domain) p.dom[c] = live;
        for (uint32_t q = 0; q < p.nq; q++) {
            if (!mark[q]) continue;
            if (!full_domain && !p.dead[q]) p.dom[c].push_back(uint16_t(q));
            if (!p.dead_user[q]) {
                p.xlat[c].push_back(full_domain ? full_idx[q] : uint16_t(p.dom[c].size() - 1));
                p.dom_user[c].push_back(uint16_t(q));
            }
        }
        if (b < ns) p.imax_user = std::max<uint32_t>(p.imax_user, uint32_t(p.dom_user[c].size()));
    }
    p.dom[p.nclass] = {q0};
    p.imax_user_stride = std::max<uint32_t>(1, p.imax_user);
    p.imax = 1;
    for (uint32_t c = 0; c <= p.nclass; c++)
        p.imax = std::max<uint32_t>(p.imax, uint32_t(p.dom[c].size()));

    // table placement
    uint32_t base = 0, defc = 0;
    uint32_t W = find_window(p, base, defc);
    auto window_words_u16 = [&](uint32_t cols) {
        uint32_t w = (cols + 1) / 2;
        if (!(w & 1)) w++;
        return w;
    };
    auto window_words_u8 = [&](uint32_t cols) {
        uint32_t w = (cols + 3) / 4;
        if (!(w & 1)) w++;
        return w;
    };
    const int fm = forced_mode;  // DFA_CREATE_TABLE_MODE (tests, layout experiments)
    if (fm == kIdentU16 && (size_t)p.nq * 512 <= smem_budget) {
        p.mode = kIdentU16;
        p.stride = 256;
    } else if (fm == kPacked9 && p.nq <= 512) {
        p.mode = kPacked9;
        p.stride = 87;
    } else if (fm == kRepU8x4 && p.nq <= u8_state_limit && (size_t)p.nq * 1024 + 1024 <= rep_budget) {
        p.mode = kRepU8x4;
        p.stride = 256;
    } else if ((fm == kRepU8x8 || (fm == 0 && p.nq >= 32)) && p.nq <= u8_state_limit &&
               (size_t)p.nq * 2048 + 2048 <= rep_budget) {
        // eight bank-group copies: ~2.96 instead of ~3.53 shared-memory
        // wavefronts per warp gather (tools/lds_gather_bench.cu, profiles/).
        // Below 32 states the 8x table copy costs more than it saves (Tiny is
        // launch/latency bound).
        p.mode = kRepU8x8;
        p.stride = 256;
    } else if (p.nq <= u8_state_limit) {
        p.mode = fm == kIdentU8 ? kIdentU8 : kIdentU8P;
        p.stride = 256;
    } else if (W && (size_t)p.nq * window_words_u16(W + 1) * 4 <= smem_budget) {
        p.mode = kWindowU16;
        p.stride = 2 * window_words_u16(W + 1);
    } else if ((size_t)p.nq * 512 <= smem_budget) {
        p.mode = kIdentU16;
        p.stride = 256;
    } else if (p.nq <= 512 && (size_t)p.nq * 87 * 4 <= smem_budget) {
        p.mode = kPacked9;
        p.stride = 87;
    } else {
        p.mode = kGlobalU16;
        p.stride = 256;
    }
    p.win_base = base;
    p.win_w = W;

    auto col_byte = [&](uint32_t col) -> uint32_t {  // window column -> a byte of its class
        return col < W ? base + col : p.class_rep[defc];
    };
    switch (p.mode) {
    case kRepU8x8:
    case kRepU8x4:
    case kIdentU8P:
    case kIdentU8: {
        p.image.assign((size_t)p.nq * 256 / 4, 0);
        uint8_t *img = reinterpret_cast<uint8_t *>(p.image.data());
        for (size_t i = 0; i < (size_t)p.nq * 256; i++) img[i] = uint8_t(p.full[i]);
        break;
    }
    case kIdentU16: {
        p.image.assign((size_t)p.nq * 256 / 2, 0);
        std::memcpy(p.image.data(), p.full.data(), (size_t)p.nq * 256 * 2);
        break;
    }
    case kWindowU8: {
        p.stride = 4 * window_words_u8(W + 1);
        p.image.assign((size_t)p.nq * p.stride / 4, 0);
        uint8_t *img = reinterpret_cast<uint8_t *>(p.image.data());
        for (uint32_t q = 0; q < p.nq; q++)
            for (uint32_t col = 0; col <= W; col++)
                img[(size_t)q * p.stride + col] = uint8_t(p.full[(size_t)q * 256 + col_byte(col)]);
        break;
    }
    case kWindowU16: {
        p.image.assign((size_t)p.nq * p.stride / 2, 0);
        uint16_t *img = reinterpret_cast<uint16_t *>(p.image.data());
        for (uint32_t q = 0; q < p.nq; q++)
            for (uint32_t col = 0; col <= W; col++)
                img[(size_t)q * p.stride + col] = p.full[(size_t)q * 256 + col_byte(col)];
        break;
    }
    case kPacked9: {
        p.image.assign((size_t)p.nq * p.stride, 0);
        for (uint32_t q = 0; q < p.nq; q++)
            for (uint32_t c = 0; c < 256; c++)
                p.image[(size_t)q * p.stride + c / 3] |= uint32_t(p.full[(size_t)q * 256 + c]) << (9 * (c % 3));
        break;
    }
    default:
        break;
    }
    return ST_OK;
}

} // namespace dfa
