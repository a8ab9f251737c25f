/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the speculative
 * chunked DFA membership test of Ko, Jung, Han, Burgstaller (arXiv:1210.5093).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1210_5093_b200/csrc); neither side includes the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; equation / algorithm
 * names are the paper's LaTeX labels.  Every function states the passage it
 * writes out.  Readings of ambiguous passages are listed in DESIGN.md
 * ("Readings"), referenced here as R1..Rn.
 *
 * Conventions shared with the spec of the problem (not with the GPU code):
 *   delta  : row-major uint16 table, delta[q*ns + c] = delta(q, c)
 *            (the paper's 2-D transition table before SBase flattening,
 *            P:1412-1420); symbol c is input byte value c (IBase).
 *   accept : bitmap, state q accepting iff (accept[q>>3] >> (q&7)) & 1.
 *   chunks : half-open [b_k, b_{k+1}); equivalent to the inclusive
 *            StartPos..EndPos ranges of Eq.StartPosition / Eq.EndPosition
 *            (P:666-687), reading R5.
 *
 * Pinned by tests/test_oracle_pins.py (worked examples of the paper,
 * brute-force substring search, closed-form DFAs, Lemma 1).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORACLE_OK 0
#define ORACLE_BAD_SYMBOL 1
#define ORACLE_BAD_ARG 2
#define ORACLE_NOT_IN_DOMAIN 3

static int is_accepting(const uint8_t *accept, uint32_t q) {
    return (accept[q >> 3] >> (q & 7)) & 1;
}

/* ------------------------------------------------------------------------
 * Alg.seqmatch, extended transition function delta-hat
 * (P:165-181).  state <- q0; for i in 0..|x|-1: state <- delta(state, x[i]).
 * Loop shape of Listing Cmatching without the pre-scaled row
 * offsets (reading R9: raw state ids, same semantics).
 * Returns ORACLE_BAD_SYMBOL if some byte >= ns (reading R12).
 * ------------------------------------------------------------------------ */
int oracle_run(const uint16_t *delta, uint32_t nq, uint32_t ns, uint16_t q0,
               const uint8_t *x, uint64_t n, uint16_t *final_state) {
    (void)nq;
    uint32_t state = q0;
    for (uint64_t i = 0; i < n; i++) {
        uint32_t c = x[i];
        if (c >= ns) return ORACLE_BAD_SYMBOL;
        state = delta[(uint64_t)state * ns + c];
    }
    *final_state = (uint16_t)state;
    return ORACLE_OK;
}

/* Alg.seqmatch line 4-6: accept iff final state in F. */
int oracle_accepts(const uint8_t *accept, uint16_t state) {
    return is_accepting(accept, state);
}

/* ------------------------------------------------------------------------
 * Same sequential run, additionally recording delta-hat(q0, x[0:pos[i]]) for
 * a sorted list of positions (the true initial state of the chunk starting
 * at pos[i]; used for the "start state in I_sigma" soundness check of
 * P:953-955).  pos must be non-decreasing and <= n.
 * ------------------------------------------------------------------------ */
int oracle_run_record(const uint16_t *delta, uint32_t nq, uint32_t ns,
                      uint16_t q0, const uint8_t *x, uint64_t n,
                      const uint64_t *pos, uint32_t npos,
                      uint16_t *state_at_pos, uint16_t *final_state) {
    (void)nq;
    uint32_t state = q0;
    uint32_t k = 0;
    for (uint64_t i = 0; i <= n; i++) {
        while (k < npos && pos[k] == i) state_at_pos[k++] = (uint16_t)state;
        if (i == n) break;
        uint32_t c = x[i];
        if (c >= ns) return ORACLE_BAD_SYMBOL;
        state = delta[(uint64_t)state * ns + c];
    }
    if (k != npos) return ORACLE_BAD_ARG;
    *final_state = (uint16_t)state;
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------
 * Error (sink) states.  The paper assumes "a unique error (or sink) state"
 * q_E that, once reached, is never left.
 * Reading R1: Z = { q not in F : delta(q, c) = q for every symbol c }.
 * dead[q] = 1 iff q in Z.  Returns |Z|.
 * ------------------------------------------------------------------------ */
uint32_t oracle_error_states(const uint16_t *delta, uint32_t nq, uint32_t ns,
                             const uint8_t *accept, uint8_t *dead) {
    uint32_t count = 0;
    for (uint32_t q = 0; q < nq; q++) {
        int absorbing = 1;
        for (uint32_t c = 0; c < ns; c++)
            if (delta[(uint64_t)q * ns + c] != q) { absorbing = 0; break; }
        dead[q] = (uint8_t)(absorbing && !is_accepting(accept, q));
        count += dead[q];
    }
    return count;
}

/* ------------------------------------------------------------------------
 * Initial-state set I_sigma, Eq.istates:
 *     I_sigma = { s : delta(x, sigma) = s }, for all s, x in Q,
 * computed as Alg.MatchingInitialStates lines 1-7, which
 * leaves out the error state (line 5; reading R1: all of Z).
 * Output sorted ascending (reading R7).  Returns |I_sigma|.
 * ------------------------------------------------------------------------ */
uint32_t oracle_initial_states(const uint16_t *delta, uint32_t nq, uint32_t ns,
                               const uint8_t *dead, uint32_t sigma,
                               uint16_t *out) {
    uint8_t *member = (uint8_t *)calloc(nq, 1);
    for (uint32_t s = 0; s < nq; s++) {                 /* foreach s in Q   */
        uint32_t target = delta[(uint64_t)s * ns + sigma]; /* delta(s, sigma) */
        if (!dead[target]) member[target] = 1;           /* if target != q_E */
    }
    uint32_t count = 0;
    for (uint32_t q = 0; q < nq; q++)
        if (member[q]) out[count++] = (uint16_t)q;
    free(member);
    return count;
}

/* Eq.MaxIstates: I_max = max over sigma of |I_sigma|. */
uint32_t oracle_imax(const uint16_t *delta, uint32_t nq, uint32_t ns,
                     const uint8_t *dead) {
    uint16_t *buf = (uint16_t *)malloc(sizeof(uint16_t) * (nq ? nq : 1));
    uint32_t best = 0;
    for (uint32_t sigma = 0; sigma < ns; sigma++) {
        uint32_t c = oracle_initial_states(delta, nq, ns, dead, sigma, buf);
        if (c > best) best = c;
    }
    free(buf);
    return best;
}

/* ------------------------------------------------------------------------
 * Multi-symbol reverse lookahead, Eq.istatesm as in
 * Alg.TwoSymISet generalised to r symbols:
 *     I_{s1..sr} = U_{q in Q} delta-hat(q, s1..sr) \ {q_E}
 * (symbols numbered in matching order).  Returns the count.
 * ------------------------------------------------------------------------ */
uint32_t oracle_initial_states_r(const uint16_t *delta, uint32_t nq,
                                 uint32_t ns, const uint8_t *dead,
                                 const uint8_t *syms, uint32_t r,
                                 uint16_t *out) {
    uint8_t *member = (uint8_t *)calloc(nq, 1);
    for (uint32_t q = 0; q < nq; q++) {
        uint32_t s = q;
        for (uint32_t i = 0; i < r; i++) s = delta[(uint64_t)s * ns + syms[i]];
        if (!dead[s]) member[s] = 1;
    }
    uint32_t count = 0;
    for (uint32_t q = 0; q < nq; q++)
        if (member[q]) out[count++] = (uint16_t)q;
    free(member);
    return count;
}

/* ------------------------------------------------------------------------
 * Input partitioning, Eq.Weights, Eq.LZero,
 * Eq.StartPosition, Eq.EndPosition, with the number
 * of states to match m = |Q| (Alg.basicmatch) or m = I_max
 * (Eq.SpeedupIStates).
 *
 *   capacities  M_k  (symbols/us), k = 0..P-1
 *   w_k = M_k / ((1/P) sum_i M_i)                                (Eq.Weights)
 *   l_0 = n*m / (w_0*m + sum_{1<=i<P} w_i)                        (Eq.LZero)
 *   Start(C_0) = 0,
 *   Start(C_k) = floor(l_0*w_0 + (1/m) sum_{1<=i<k} l_0*w_i)      k >= 1
 *   End(C_k)   = n-1 for k = P-1, else Start(C_{k+1}) - 1
 *
 * All arithmetic is exact rational arithmetic on 128-bit integers (reading
 * R4: exact floor, never floating point).  Each rational is kept as
 * numerator/denominator in the order the paper writes the terms.
 * Output: start[k] for k=0..P-1 and start[P] = n (half-open bounds).
 * Returns ORACLE_BAD_ARG for P == 0, m == 0 or a zero capacity.
 * ------------------------------------------------------------------------ */
typedef unsigned __int128 u128;

int oracle_chunk_bounds(uint64_t n, uint32_t P, uint32_t m,
                        const uint64_t *capacity, uint64_t *bounds) {
    if (P == 0 || m == 0) return ORACLE_BAD_ARG;
    u128 sumM = 0;
    for (uint32_t i = 0; i < P; i++) {
        if (capacity[i] == 0) return ORACLE_BAD_ARG;
        sumM += capacity[i];
    }
    /* w_k = wnum_k / wden with wnum_k = P*M_k, wden = sum M.             */
    u128 wden = sumM;
    /* l_0 = n*m / (w_0*m + sum_{i>=1} w_i)
     *     = n*m*wden / (wnum_0*m + sum_{i>=1} wnum_i)                    */
    u128 den_inner = (u128)P * capacity[0] * m;
    for (uint32_t i = 1; i < P; i++) den_inner += (u128)P * capacity[i];
    u128 l0_num = (u128)n * m * wden;
    u128 l0_den = den_inner;
    bounds[0] = 0;
    u128 sum_wnum = 0;                  /* sum_{1<=i<k} wnum_i, running sum */
    for (uint32_t k = 1; k < P; k++) {
        /* l_0*w_0 = l0_num*wnum_0 / (l0_den*wden)                         */
        /* (1/m) sum_{1<=i<k} l_0*w_i = l0_num*sum wnum_i / (m*l0_den*wden) */
        if (k >= 2) sum_wnum += (u128)P * capacity[k - 1];
        u128 common_den = (u128)m * l0_den * wden;
        u128 term0 = l0_num * ((u128)P * capacity[0]) * m; /* over common_den */
        u128 term1 = l0_num * sum_wnum;                       /* over common_den */
        bounds[k] = (uint64_t)((term0 + term1) / common_den);
    }
    bounds[P] = n;
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------
 * State map of one chunk: L_i[j] = delta-hat(q_j, C_i), taken
 * over the initial-state set of the chunk's reverse lookahead symbol
 * sigma = x[b_k - 1] (Alg.MatchingInitialStates lines 17-19).
 * row[j] for j < |I_sigma| in ascending state order; row[j] = 0xFFFF for
 * |I_sigma| <= j < row_len (reading R6: non-domain slots are never read).
 * Returns ORACLE_BAD_SYMBOL on a byte >= ns.
 * ------------------------------------------------------------------------ */
int oracle_chunk_map(const uint16_t *delta, uint32_t nq, uint32_t ns,
                     const uint8_t *dead, const uint8_t *x, uint64_t n,
                     uint64_t begin, uint64_t end, uint32_t row_len,
                     uint16_t *row, uint32_t *domain_size) {
    if (begin == 0 || begin > end || end > n) return ORACLE_BAD_ARG;
    uint32_t sigma = x[begin - 1];                 /* reverse lookahead symbol */
    if (sigma >= ns) return ORACLE_BAD_SYMBOL;
    uint16_t *I = (uint16_t *)malloc(sizeof(uint16_t) * (nq ? nq : 1));
    uint32_t count = oracle_initial_states(delta, nq, ns, dead, sigma, I);
    if (count > row_len) { free(I); return ORACLE_BAD_ARG; }
    for (uint32_t j = 0; j < row_len; j++) row[j] = 0xFFFF;
    for (uint32_t j = 0; j < count; j++) {         /* foreach j in I_{C_i}   */
        uint32_t state = I[j];
        for (uint64_t p = begin; p < end; p++) {  /* for k <- Start to End  */
            uint32_t c = x[p];
            if (c >= ns) { free(I); return ORACLE_BAD_SYMBOL; }
            state = delta[(uint64_t)state * ns + c];
        }
        row[j] = (uint16_t)state;
    }
    free(I);
    if (domain_size) *domain_size = count;
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------
 * Chunk map with r reverse lookahead symbols (Sec. "Multiple Reverse
 * Lookahead Symbols"): the domain of chunk [begin, end) is
 * I_{s1..sL} of Eq.istatesm for the L = min(r, begin) symbols before it,
 * s1..sL = x[begin-L .. begin-1] in matching order; the row
 * holds delta-hat(q, x[begin..end)) for every q of that domain (ascending),
 * dom receives the domain.  Unused entries of both are 0xFFFF.
 * ------------------------------------------------------------------------ */
int oracle_chunk_map_r(const uint16_t *delta, uint32_t nq, uint32_t ns,
                       const uint8_t *dead, const uint8_t *x, uint64_t n,
                       uint64_t begin, uint64_t end, uint32_t r,
                       uint32_t row_len, uint16_t *dom, uint16_t *row,
                       uint32_t *domain_size) {
    if (begin == 0 || begin > end || end > n || r == 0) return ORACLE_BAD_ARG;
    uint32_t L = (uint64_t)r < begin ? r : (uint32_t)begin;
    const uint8_t *syms = x + (begin - L);
    for (uint32_t i = 0; i < L; i++)
        if (syms[i] >= ns) return ORACLE_BAD_SYMBOL;
    uint16_t *I = (uint16_t *)malloc(sizeof(uint16_t) * (nq ? nq : 1));
    uint32_t count = oracle_initial_states_r(delta, nq, ns, dead, syms, L, I);
    if (count > row_len) { free(I); return ORACLE_BAD_ARG; }
    for (uint32_t j = 0; j < row_len; j++) { row[j] = 0xFFFF; dom[j] = 0xFFFF; }
    for (uint32_t j = 0; j < count; j++) {         /* foreach q in I_{s1..sL} */
        uint32_t state = I[j];
        for (uint64_t p = begin; p < end; p++) {  /* for k <- Start to End   */
            uint32_t c = x[p];
            if (c >= ns) { free(I); return ORACLE_BAD_SYMBOL; }
            state = delta[(uint64_t)state * ns + c];
        }
        dom[j] = I[j];
        row[j] = (uint16_t)state;
    }
    free(I);
    if (domain_size) *domain_size = count;
    return ORACLE_OK;
}

/* All maps of a partition, chunks 1..P-1 (chunk 0 yields only its end state,
 * P:803-804, 1062-1066), run in parallel over chunks with plain pthreads --
 * the "forpar" of Alg.MatchingInitialStates line 8.  maps has
 * (P-1)*row_len entries, row k-1 = chunk k.  chunk0_end = delta-hat(q0,C_0). */
typedef struct {
    const uint16_t *delta; uint32_t nq, ns; const uint8_t *dead;
    const uint8_t *x; uint64_t n; const uint64_t *bounds; uint32_t P;
    uint32_t row_len; uint16_t *maps; uint32_t next; pthread_mutex_t *lock;
    int status;
} maps_job;

static void *maps_worker(void *arg) {
    maps_job *job = (maps_job *)arg;
    for (;;) {
        pthread_mutex_lock(job->lock);
        uint32_t k = job->next++;
        pthread_mutex_unlock(job->lock);
        if (k >= job->P) break;
        int st = oracle_chunk_map(job->delta, job->nq, job->ns, job->dead,
                                  job->x, job->n, job->bounds[k],
                                  job->bounds[k + 1], job->row_len,
                                  job->maps + (uint64_t)(k - 1) * job->row_len,
                                  NULL);
        if (st != ORACLE_OK) {
            pthread_mutex_lock(job->lock);
            if (job->status == ORACLE_OK) job->status = st;
            pthread_mutex_unlock(job->lock);
        }
    }
    return NULL;
}

int oracle_maps(const uint16_t *delta, uint32_t nq, uint32_t ns,
                const uint8_t *dead, uint16_t q0, const uint8_t *x, uint64_t n,
                const uint64_t *bounds, uint32_t P, uint32_t row_len,
                uint32_t threads, uint16_t *chunk0_end, uint16_t *maps) {
    if (P == 0 || bounds[0] != 0 || bounds[P] != n) return ORACLE_BAD_ARG;
    int st = oracle_run(delta, nq, ns, q0, x, bounds[1 <= P ? 1 : 0],
                        chunk0_end);                 /* chunk C_0 from q0 */
    if (st != ORACLE_OK) return st;
    if (P == 1) return ORACLE_OK;
    if (threads == 0) threads = 1;
    pthread_mutex_t lock;
    pthread_mutex_init(&lock, NULL);
    maps_job job = {delta, nq, ns, dead, x, n, bounds, P, row_len, maps, 1,
                    &lock, ORACLE_OK};
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    for (uint32_t t = 0; t < threads; t++)
        pthread_create(&tid[t], NULL, maps_worker, &job);
    for (uint32_t t = 0; t < threads; t++) pthread_join(tid[t], NULL);
    free(tid);
    pthread_mutex_destroy(&lock);
    return job.status;
}

/* ------------------------------------------------------------------------
 * Sequential merge, Eq.SeqReduction:
 *     last = L_{P-1}[ L_{P-2}[ ... L_0[0] ... ] ]
 * where indexing L_k by a state means "the entry of that state in I_sigma_k".
 * A state in Z stays where it is (the error state is never left,
 * P:450-454; reading R1).  A state neither in Z nor in I_sigma_k would mean
 * the speculation was unsound: ORACLE_NOT_IN_DOMAIN.
 * ------------------------------------------------------------------------ */
int oracle_fold(const uint16_t *delta, uint32_t nq, uint32_t ns,
                const uint8_t *dead, const uint8_t *x, const uint64_t *bounds,
                uint32_t P, uint32_t row_len, uint16_t chunk0_end,
                const uint16_t *maps, uint16_t *final_state) {
    uint16_t *I = (uint16_t *)malloc(sizeof(uint16_t) * (nq ? nq : 1));
    uint32_t state = chunk0_end;
    for (uint32_t k = 1; k < P; k++) {
        if (dead[state]) continue;
        uint32_t sigma = x[bounds[k] - 1];
        uint32_t count = oracle_initial_states(delta, nq, ns, dead, sigma, I);
        uint32_t j = 0;
        while (j < count && I[j] != state) j++;
        if (j == count) { free(I); return ORACLE_NOT_IN_DOMAIN; }
        state = maps[(uint64_t)(k - 1) * row_len + j];
    }
    free(I);
    *final_state = (uint16_t)state;
    return ORACLE_OK;
}

/* Binary combining operation of Eq.MapReduction on dense maps
 * over Q: Lij[q] = Lj[Li[q]].  Pinned by the hand-derived dense maps of
 * Fig.motivDFA (L_{0,1,2}[q0] = q1, tests/golden/fig_motiv_dfa.json) and by
 * compose(M(u), M(v)) == M(uv) against Alg.seqmatch runs. */
void oracle_compose_dense(const uint16_t *Li, const uint16_t *Lj, uint32_t nq,
                          uint16_t *Lij) {
    for (uint32_t q = 0; q < nq; q++) Lij[q] = Lj[Li[q]];
}
