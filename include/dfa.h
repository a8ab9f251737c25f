/*
 * dfa.h -- C ABI of the B200 speculative chunked DFA membership test
 * (Ko, Jung, Han, Burgstaller, arXiv:1210.5093).
 *
 * Citations "P:n" are lines of the paper's LaTeX source; names in
 * CamelCase/dots are its \label{}s.  The library is libdfa.so, built from
 * paper_1210_5093_b200/csrc.  No C++ or torch types cross this boundary:
 * plain integers and pointers only.  A CUDA stream is passed as `void*`
 * (a cudaStream_t; NULL = the legacy default stream).
 *
 * Problem (Alg.seqmatch): given a DFA
 * (Q, Sigma, delta, q0, F) and an input x, compute delta-hat(q0, x) and
 * whether it is in F.  The library computes it as the paper does:
 * the input is partitioned into chunks (Eq.LZero / Eq.StartPosition /
 * Eq.EndPosition), every chunk k >= 1 is matched speculatively
 * from the initial-state set I_sigma of its reverse-lookahead symbol
 * sigma = x[b_k - 1] (Eq.istates, Alg.MatchingInitialStates
 * P:1031-1079), each chunk yields a state map L_k, and the maps
 * are composed (Eq.SeqReduction, Eq.MapReduction).
 *
 * Conventions (readings R1-R12 in DESIGN.md):
 *  - symbols are input bytes: byte b is column b of the table; a byte
 *    >= alphabet_size is an error (DFA_ERR_SYMBOL), reading R12;
 *  - error states Z = { q not in F : delta(q,c) = q for all c } (the paper's
 *    q_E), reading R1.  I_sigma = delta(Q, sigma) \ Z
 *    (Alg.MatchingInitialStates line 5), listed in ascending order;
 *  - I_max = max over sigma < alphabet_size of |I_sigma| (Eq.MaxIstates);
 *    it is the row stride of the map arrays (at least 1);
 *  - chunks are half-open [b_k, b_{k+1}), b_0 = 0, b_P = n (R5);
 *  - the chunk-0 length ratio c = c_num/c_den replaces the paper's
 *    w_0*m/w (Eq.LZero with homogeneous w_i, i >= 1):
 *        b_k = floor(n * (c + k - 1) / (c + P - 1)),  1 <= k <= P-1,
 *    evaluated exactly in integers (R3, R4);
 *  - state maps are compact: row k-1 (chunk k >= 1) has entry
 *    j = delta-hat(I_sigma_k[j], C_k) for j < |I_sigma_k| and 0xFFFF after
 *    (R6, R7).  Chunk 0 yields the single state e0 = delta-hat(q0, C_0) (R8).
 *
 * Ownership: dfa_create copies the table and bitmap (the caller may free
 * them on return).  The handle owns its device copies and scratch, freed by
 * dfa_destroy.  Device footprint of a handle: the tables (|Q| x 256 uint16, the
 * I_sigma lists and rank tables over the byte classes), for I_max > 8 the
 * two-symbol sets of Eq.istatesm (classes^2 x max |I_{s1 s2}| x 4 bytes, built
 * only up to 128 MiB), and scratch that grows with the largest call (about
 * 2 x I_max bytes per execution sub-chunk, ~10^5 sub-chunks).  Every dev_* pointer is caller-owned device memory, borrowed
 * for the stream-ordered lifetime of the call.
 *
 * Errors: every call returns a dfa_status; nothing is thrown across the
 * ABI; out-parameters are untouched on error.  Calls on one handle must not
 * overlap in time (one in-flight call per handle; it owns one scratch area).
 */
#ifndef DFA_H
#define DFA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dfa_handle *dfa_handle_t;

typedef enum {
    DFA_OK = 0,
    DFA_ERR_ARG = 1,       /* NULL pointer, bad option, host-only handle used for compute */
    DFA_ERR_STATES = 2,    /* |Q| == 0 or > 65000, q0 >= |Q|, table entry >= |Q| */
    DFA_ERR_ALPHABET = 3,  /* |Sigma| == 0 or > 256 */
    DFA_ERR_CHUNKS = 4,    /* P == 0, n < c + P - 1, or explicit bounds not strictly increasing */
    DFA_ERR_SYMBOL = 5,    /* an input byte >= |Sigma| */
    DFA_ERR_OOM = 6,       /* device or host allocation failed */
    DFA_ERR_CUDA = 7,      /* a CUDA runtime call failed (no device, launch failure) */
    DFA_ERR_INTERNAL = 8   /* a device-side consistency check failed (bug) */
} dfa_status;

/* Static analysis of a DFA (host preprocessing at dfa_create). */
typedef struct {
    uint32_t num_states;      /* |Q| */
    uint32_t alphabet_size;   /* |Sigma| */
    uint32_t num_classes;     /* distinct table columns over 0..|Sigma|-1 */
    uint32_t i_max;           /* Eq.MaxIstates, >= 1; map row stride */
    uint32_t gamma_num;       /* gamma = I_max / |Q \ Z| (Eq.obtained_speedup, R2) */
    uint32_t gamma_den;
    uint32_t num_dead;        /* |Z| */
    uint32_t dead_state;      /* smallest state of Z, 0xFFFF if Z is empty */
    uint32_t num_absorbing;   /* states with delta(q,c) = q for all c (incl. accepting) */
    uint32_t table_mode;      /* device table layout, DFA_TABLE_* */
    uint32_t table_bytes;     /* bytes of the device table kept in shared memory (0 = global) */
    uint32_t c_num, c_den;    /* chunk-0 length ratio c used by dfa_chunk_maps */
    uint32_t device_ready;    /* 1 if device tables were uploaded (0 = host-only handle) */
} dfa_info;

enum {
    DFA_TABLE_IDENT_U8 = 1,   /* smem, 256 byte-indexed columns, uint8 states   */
    DFA_TABLE_IDENT_U16 = 2,  /* smem, 256 byte-indexed columns, uint16 states  */
    DFA_TABLE_WINDOW_U8 = 3,  /* smem, columns = byte window + default column  */
    DFA_TABLE_WINDOW_U16 = 4,
    DFA_TABLE_PACKED9 = 5,    /* smem, 9-bit states packed 3 per 32-bit word    */
    DFA_TABLE_GLOBAL_U16 = 6, /* global memory through L1/__ldg                 */
    DFA_TABLE_REP8_U8 = 7,    /* smem, IDENT_U8 image x 8 copies, copy g in banks
                                 4g..4g+3, read by lanes l = g mod 8 (32..110 states) */
    DFA_TABLE_REP4_U8 = 8,    /* same with 4 copies (only when forced)          */
    DFA_TABLE_IDENT_U8_PAD = 9 /* smem, uint8 states, rows of 260 bytes: entry
                                 (s, b) in bank (s + b/4) mod 32 (<= 252 states) */
};

/* dfa_create_ex flags */
enum {
    DFA_CREATE_HOST_ONLY = 1,  /* analysis only: no device memory touched; compute calls fail */
    DFA_CREATE_FULL_DOMAIN = 2 /* Alg.2 ablation: every sub-chunk matched from all of
                                  Q \ Z instead of I_sigma; results identical, i_max unchanged
                                  (API rows stay over I_sigma), speed shows the I_sigma win */
};
/* Force a shared-memory table layout (a DFA_TABLE_* value) instead of the
 * default choice: flags |= DFA_CREATE_TABLE_MODE(m).  Used by the layout parity
 * tests and the layout experiments; a layout that cannot hold the DFA falls back
 * to the default choice (dfa_get_info reports the layout taken). */
#define DFA_CREATE_TABLE_MODE(m) (((uint32_t)(m) & 0xFu) << 8)

/*
 * dfa_create: validate and analyse a DFA, upload device tables.
 *   table          host, |Q|*|Sigma| uint16, table[q*|Sigma| + c] = delta(q, c)
 *   num_states     |Q|, 1..65000
 *   alphabet_size  |Sigma|, 1..256; input byte b is symbol b
 *   q0             start state
 *   accept_bitmap  host, ceil(|Q|/8) bytes; q in F iff bit (q&7) of byte q>>3
 *   out            receives the handle
 * Host work O(|Q|*256): error states, column classes, I_sigma for every
 * symbol (Alg.MatchingInitialStates lines 1-7, computed once
 * offline as P:1099-1103 allows), I_max, gamma, table placement.
 */
dfa_status dfa_create(const uint16_t *table, uint32_t num_states, uint32_t alphabet_size,
                      uint16_t q0, const uint8_t *accept_bitmap, dfa_handle_t *out);
dfa_status dfa_create_ex(const uint16_t *table, uint32_t num_states, uint32_t alphabet_size,
                         uint16_t q0, const uint8_t *accept_bitmap, uint32_t flags,
                         dfa_handle_t *out);
dfa_status dfa_destroy(dfa_handle_t h);

dfa_status dfa_get_info(dfa_handle_t h, dfa_info *out);

/* I_sigma for symbol `sigma` (ascending); out_states must hold i_max entries. */
dfa_status dfa_domain(dfa_handle_t h, uint32_t sigma, uint16_t *out_states, uint32_t *out_count);

/* Chunk-0 length ratio c = c_num/c_den (both 1..2^20) used by dfa_chunk_maps. */
dfa_status dfa_set_chunk_ratio(dfa_handle_t h, uint32_t c_num, uint32_t c_den);

/* Host evaluation of the partition formula (above) into host_bounds[P+1]. */
dfa_status dfa_plan_bounds(uint64_t n, uint32_t num_chunks, uint32_t c_num, uint32_t c_den,
                           uint64_t *host_bounds);

/*
 * dfa_match: membership test of dev_input[0..len) (device memory).  Runs the
 * chunked speculative path on `stream` and synchronises it to return host
 * scalars: *final_state = delta-hat(q0, x), *accept = (final in F).
 * len == 0 returns (q0, F[q0]) without launching.  DFA_ERR_SYMBOL if some
 * byte >= |Sigma|.
 */
dfa_status dfa_match(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, void *stream,
                     uint16_t *final_state, int *accept);

/*
 * dfa_match_host: the same call for an input in HOST memory (pinned for
 * full speed; the handle keeps a device copy buffer of len bytes).  Inputs
 * longer than one piece (DFA_OPT_HOST_PIECE, default 32 MiB) are pipelined:
 * piece g+1 is copied on an internal stream while piece g is matched on
 * `stream` as a segment map (dfa_segment_map) folded into the running state.
 * Early exit (DFA_OPT_EARLY_EXIT, default on): once
 * a finished piece leaves the run in a state that absorbs every byte (an
 * absorbing accept of a suffix-closed language, or an error state), the
 * remaining pieces are neither copied nor matched -- the result cannot
 * change.  Synchronises `stream`; dfa_get_stats().host_bytes = bytes copied.
 */
dfa_status dfa_match_host(dfa_handle_t h, const uint8_t *host_input, uint64_t len, void *stream,
                          uint16_t *final_state, int *accept);

/*
 * dfa_chunk_maps: the per-chunk results for P = num_chunks reporting chunks
 * with the handle's c (asynchronous on `stream`; DFA_ERR_CHUNKS if
 * len < c + P - 1 so that some chunk would be empty):
 *   dev_bounds      [P+1]  uint64 chunk offsets (out)
 *   dev_chunk0_end  [1]    e0 = delta-hat(q0, C_0) (out)
 *   dev_maps        [(P-1)*i_max] uint16 compact maps (out; may be NULL iff P == 1)
 *   dev_chunk_start [P]    true initial state of every chunk (out; may be NULL)
 *   dev_final       [2]    {final state, accept} as uint16 (out; may be NULL)
 * A bad symbol is reported by dfa_get_last_device_error after a stream sync.
 */
dfa_status dfa_chunk_maps(dfa_handle_t h, const uint8_t *dev_input, uint64_t len,
                          uint32_t num_chunks, void *stream, uint64_t *dev_bounds,
                          uint16_t *dev_chunk0_end, uint16_t *dev_maps,
                          uint16_t *dev_chunk_start, uint16_t *dev_final);

/* Same for a caller-given partition dev_bounds_in[P+1] (device memory):
 * 0 = b_0 < b_1 < ... < b_P = len, validated on the host after a copy. */
dfa_status dfa_chunk_maps_at(dfa_handle_t h, const uint8_t *dev_input, uint64_t len,
                             uint32_t num_chunks, const uint64_t *dev_bounds_in, void *stream,
                             uint16_t *dev_chunk0_end, uint16_t *dev_maps,
                             uint16_t *dev_chunk_start, uint16_t *dev_final);

/*
 * dfa_match_batch: many independent inputs in one pass (multi-input
 * batching; the paper packs inputs and automata into one SBase/IBase layout,
 * P:1430-1440).  Input j is dev_data[dev_offsets[j] .. dev_offsets[j+1])
 * (device bytes, data_len of them; dev_offsets: DEVICE array of count+1
 * non-decreasing offsets <= data_len), each matched from q0 as its own
 * membership test (Alg.seqmatch).  Writes dev_final[j] (uint16 final state)
 * and dev_accept[j] (uint8 0/1), device arrays of count entries; empty inputs
 * give (q0, F[q0]).  Inside, the inputs are the reporting chunks of one
 * partition whose chunks all start from {q0} (no speculation across inputs,
 * no fold).  count >= 4096: fully asynchronous, one sub-chunk per input, bad
 * offsets are clamped and reported as DFA_ERR_ARG by
 * dfa_get_last_device_error; count < 4096: the offsets are read back (the
 * call synchronises `stream` once), validated (DFA_ERR_ARG) and each input is
 * split for parallelism.  A byte >= |Sigma| is reported by
 * dfa_get_last_device_error.
 */
dfa_status dfa_match_batch(dfa_handle_t h, const uint8_t *dev_data, uint64_t data_len, const uint64_t *dev_offsets,
                           uint32_t count, void *stream, uint16_t *dev_final, uint8_t *dev_accept);

/*
 * dfa_lookahead_maps: multiple reverse lookahead symbols (PAPER.md Sec.
 * "Multiple Reverse Lookahead Symbols"; Eq.istatesm P:1142-1147,
 * Alg.TwoSymISet).  Restricts the maps of a preceding
 * dfa_chunk_maps(_at) call (same stream, same input and partition) to the
 * r-symbol initial-state sets.  For chunk k = 1..P-1, with L = min(r, b_k)
 * and s1..sL = x[b_k-L .. b_k-1] (matching order):
 *   dev_domains[(k-1)*i_max + i] = i-th state of I_{s1..sL} = delta-hat(Q, s1..sL) \ Z (ascending)
 *   dev_maps_r [(k-1)*i_max + i] = delta-hat(that state, C_k), taken from dev_maps
 *                                  (Lemma 1: I_{s1..sL} is a subset of I_{sL})
 *   dev_domain_sizes[k-1]        = |I_{s1..sL}|
 * Unused entries are 0xFFFF.  Inputs (device): dev_input[len], dev_bounds[P+1]
 * and dev_maps[(P-1)*i_max] as written by the chunk-maps call; outputs
 * (device): dev_domains and dev_maps_r [(P-1)*i_max], dev_domain_sizes[P-1].
 * r = 1..16 (r = 1 reproduces I_sigma).  P == 1: nothing to do.  Asynchronous;
 * a lookahead byte >= |Sigma| is reported by dfa_get_last_device_error.
 * O(r |Q|) table reads per chunk.
 */
dfa_status dfa_lookahead_maps(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, uint32_t num_chunks,
                              const uint64_t *dev_bounds, const uint16_t *dev_maps, uint32_t r, void *stream,
                              uint16_t *dev_domains, uint16_t *dev_domain_sizes, uint16_t *dev_maps_r);

/*
 * Multi-GPU sharding (the paper's two-tier merge, Fig.Merge
 * P:1530-1647, with NVLink in place of MPI).  A segment g of a longer input
 * x = x_0 x_1 ... x_{G-1} is matched on its own GPU:
 * dfa_segment_map writes dev_row[i_max] = the composed map of the segment over
 * I_sigma of `lookahead` = the last byte of segment g-1 (ascending, 0xFFFF
 * padded), or, for lookahead = -1 (segment 0), dev_row[0] = delta-hat(q0, x_0).
 * After the G rows are gathered (one allgather of G*i_max uint16),
 * dfa_fold_segments folds them in order (Eq.SeqReduction) into dev_final =
 * {final state, accept} (asynchronous; errors via dfa_get_last_device_error).
 * dev_lookahead[g] (device, G bytes) = last byte of segment g-1 (entry 0 unused).
 */
dfa_status dfa_segment_map(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, int32_t lookahead,
                           void *stream, uint16_t *dev_row);
/*
 * dfa_segment_chunk_maps: the per-GPU step of the sharded path with the same
 * partition and kernels as dfa_chunk_maps.  The segment (dev_input, len) is cut
 * into num_chunks chunks (c-form, dfa_set_chunk_ratio); chunk 0 is matched from
 * {q0} (lookahead = -1: the segment starts the string) or from I_sigma of
 * sigma = lookahead (the byte before the segment, Eq.istates).
 * Outputs (caller-owned device memory; asynchronous on `stream`):
 *   dev_bounds       [num_chunks+1] uint64 chunk bounds (may be NULL)
 *   dev_chunk0_row   lookahead = -1: [1] = e0 = delta-hat(q0, C_0); else
 *                    [i_max] = chunk 0's map over the user's I_sigma (ascending, 0xFFFF padded)
 *   dev_maps         [(num_chunks-1) * i_max] rows of chunks 1.., as dfa_chunk_maps
 *   dev_segment_row  [i_max] the composed map of the whole segment over chunk 0's
 *                    domain (Eq.MapReduction), i.e. the dfa_segment_map row; for
 *                    lookahead = -1 entry 0 is the segment's final state
 * Repeated identical calls replay a captured CUDA graph; the partition stays on
 * the device (no host round trip per call).  Errors as dfa_chunk_maps, plus
 * DFA_ERR_SYMBOL for lookahead >= |Sigma|.
 */
dfa_status dfa_segment_chunk_maps(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, uint32_t num_chunks,
                                  int32_t lookahead, void *stream, uint64_t *dev_bounds,
                                  uint16_t *dev_chunk0_row, uint16_t *dev_maps, uint16_t *dev_segment_row);
dfa_status dfa_fold_segments(dfa_handle_t h, const uint16_t *dev_rows, const uint8_t *dev_lookahead,
                             uint32_t G, void *stream, uint16_t *dev_final);

/*
 * Measurement aid (not part of the method): the match kernel's step alone.
 * T = *out_threads threads each run ONE lane from q0 over their own
 * *out_per_thread consecutive bytes of dev_input (a multiple of 32; the first
 * T * per bytes are used) with the handle's table layout, load pattern and
 * 16-byte block step, and none of the method's bookkeeping (domains I_sigma,
 * convergence checks, maps, composition).  Its throughput is the practical
 * ceiling of the layout on this input, reported beside the lanes kernel's
 * (bench.py roofline.lds_ceiling).  dev_out[t] (device, caller-owned, >= T
 * entries; query T first by passing dev_out = NULL) = delta-hat(q0, bytes of
 * thread t) (Alg.seqmatch over that range, checkable against the oracle).
 * dev_input must be 32-byte aligned and len >= 32 * T, else DFA_ERR_ARG.
 * Bad symbols are not detected.  Asynchronous.
 */
dfa_status dfa_gather_ceiling(dfa_handle_t h, const uint8_t *dev_input, uint64_t len, void *stream,
                              uint16_t *dev_out, uint64_t *out_per_thread, uint32_t *out_threads);

/* After a stream sync: DFA_ERR_SYMBOL / DFA_ERR_INTERNAL raised by the last
 * asynchronous call's kernels, else DFA_OK.  Clears the flag. */
dfa_status dfa_get_last_device_error(dfa_handle_t h);

/*
 * Tuning / measurement options (DFA_OPT_*).  Defaults are chosen by the
 * library from the table placement and the device's SM count.
 */
enum {
    DFA_OPT_SUBCHUNK_TARGET = 1, /* number of execution sub-chunks per call (0 = auto) */
    DFA_OPT_CONVERGENCE = 2,     /* 1 = merge converged lanes (default), 0 = off */
    DFA_OPT_PROFILE = 3,         /* 1 = record per-kernel CUDA-event times */
    DFA_OPT_THREADS_PER_CTA = 4, /* match kernel CTA size (0 = auto) */
    DFA_OPT_TREE_FANIN = 5,      /* max children per composition-tree node, 2..64 (default 32) */
    DFA_OPT_FOLD_IN_TREE = 6,    /* 1: maps of <= 16 entries go through tree_kernel (also for the final
                                    fold) instead of the rank-space compose8 / fold_rows paths */
    DFA_OPT_WARP_COMPOSE = 7,    /* 1 (default): maps of <= 8 entries composed in rank space: in the match
                                    kernel's warps, leaf_fold_kernel and compose8_kernel; 0: tree path */
    DFA_OPT_GRAPHS = 8,          /* 1 (default): replay a CUDA graph when a dfa_chunk_maps call repeats */
    DFA_OPT_MAX_LANES = 9,       /* lanes per thread in the match kernel, 1..8 (default 8): converge_kernel
                                    runs until at most this many lanes survive; larger domains without
                                    the converge stage take several passes */
    DFA_OPT_HOST_PIECE = 10,     /* dfa_match_host piece size in bytes (>= 1 MiB, default 32 MiB) */
    DFA_OPT_EARLY_EXIT = 11,     /* 1 (default): dfa_match_host stops at an absorbing running state */
    DFA_OPT_STICKY_PARKING = 12, /* 1 (default): park lanes in sticky states; 0 = off */
    DFA_OPT_COUNT_WORK = 13,     /* 1: the match kernels count the lane-steps (table lookups) they execute,
                                    summed into dfa_stats.work_* until dfa_get_stats reads them; 0 (default) */
    DFA_OPT_FUSED_TAIL = 14,     /* 1: maps of <= 8 entries are composed by the match kernel's CTAs themselves
                                    (one launch); 0 (default, measured faster): leaf_fold_kernel + compose8_kernel */
    DFA_OPT_FACTORED = 15,       /* 1 (default): maps of more than 16 entries behind the converge stage are
                                    composed in factored form (the first sub-chunk's converge map, then <= 8
                                    survivor values per node; Eq.MapReduction on the image of the first map);
                                    0: every node composes full rows (walk_kernel) */
    DFA_OPT_LOOKAHEAD2 = 16,     /* 1 (default): with the factored composition, internal execution sub-chunks
                                    start from the two-symbol initial set I_{s1 s2} (Eq.istatesm, r = 2,
                                    PAPER.md 1129-1147) instead of I_{s2}; results identical, fewer lanes */
    DFA_OPT_TMA_INPUT = 17       /* 1: where the table layout has it (rep8_u8), the match kernel stages its
                                    input through shared memory with TMA gather copies (IBase streaming,
                                    PAPER.md 1433-1440); 0 (default, measured faster): per-thread 32-byte loads */
};
dfa_status dfa_set_option(dfa_handle_t h, uint32_t key, int64_t value);

/* Statistics.  input_bytes .. num_kernels describe the last call.  With
 * DFA_OPT_PROFILE on, every call records CUDA events (on its stream) around
 * its kernel sections; dfa_get_stats synchronises them, returns the summed
 * durations per section over all calls since the previous dfa_get_stats
 * (kernel_name[i] / kernel_ms[i]; profiled = number of calls summed) and
 * resets the accumulators. */
typedef struct {
    uint64_t input_bytes;      /* n */
    uint64_t num_subchunks;    /* execution sub-chunks of the last call */
    uint32_t num_kernels;      /* kernels launched by the last call */
    uint32_t profiled;         /* calls accumulated in kernel_ms */
    float kernel_ms[8];        /* summed section durations (DFA_OPT_PROFILE) */
    char kernel_name[8][32];
    uint64_t host_bytes;       /* bytes dfa_match_host copied to the device in its last call */
    /* DFA_OPT_COUNT_WORK: executed lane-steps (one table lookup each) since the
     * previous dfa_get_stats: [0] converge_kernel, [1] lanes_kernel (including
     * the re-read of parked sticky lanes).  0 when the option is off. */
    uint64_t work_lookups[2];
    uint32_t work_calls;       /* calls summed in work_lookups */
} dfa_stats;
dfa_status dfa_get_stats(dfa_handle_t h, dfa_stats *out);

const char *dfa_status_string(dfa_status s);

/* Human-readable detail (CUDA error name, call site) of the last DFA_ERR_CUDA /
 * DFA_ERR_OOM returned on the calling thread; "" if none. */
const char *dfa_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif /* DFA_H */
