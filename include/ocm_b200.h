/*
 * ocm_b200.h — C-ABI of the B200-native optimal-cycle-mean solver.
 *
 * Plain pointers and sizes only (no C++ or torch types). Each entry point
 * replaces one reference interface (paths relative to the reference's proj/):
 *
 *   ocm_build_graph       include/ocm/graph.hpp:76      ocm::build_graph
 *   ocm_parse_graph_text  include/ocm/graph_io.hpp:41   ocm::parse_graph_text
 *   ocm_read_graph_file   include/ocm/graph_io.hpp:45   ocm::read_graph_file
 *   ocm_graph_edges       include/ocm/graph.hpp:61      Graph::edges()
 *   ocm_generate_model    include/ocm/model_gen.hpp:67  ocm::generate_model
 *   ocm_solve             include/ocm/solve.hpp:64      ocm::solve (lane howard-par)
 *   ocm_session_*         include/ocm/howard_par.hpp:90 HowardPar (state kept resident
 *                         in HBM so a graph can be solved repeatedly without re-upload)
 *
 * Error behaviour mirrors the reference's exceptions as return codes:
 * std::invalid_argument -> OCM_E_INVALID, ParseError -> OCM_E_PARSE (message
 * "<source>:<line>: <what>", line via ocm_last_error_line), std::logic_error
 * (structural: a vertex without successor in its region, lambda increase)
 * -> OCM_E_LOGIC. The message of the last failure on the calling thread is
 * returned by ocm_last_error(). There is no CPU fallback: without a usable
 * sm_100a device every solve returns OCM_E_CUDA.
 */
#ifndef OCM_B200_H
#define OCM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCM_OK 0
#define OCM_E_INVALID 1     /* std::invalid_argument */
#define OCM_E_PARSE 2       /* ocm::ParseError */
#define OCM_E_LOGIC 3       /* std::logic_error */
#define OCM_E_CUDA 4        /* no device / CUDA failure */
#define OCM_E_UNSUPPORTED 5 /* lane or option not provided by this library */
#define OCM_E_RANGE 6       /* exact arithmetic would overflow 64-bit keys */
#define OCM_E_IO 7          /* std::runtime_error from file access */

/* include/ocm/solve.hpp:21 enum Algo (only howard-par runs on the device) */
#define OCM_ALGO_HOWARD 0
#define OCM_ALGO_HOWARD_PAR 1
#define OCM_ALGO_LAWLER 2
#define OCM_ALGO_TREE 3
#define OCM_ALGO_ORACLE_ENUM 4
#define OCM_ALGO_ORACLE_DP 5
/* include/ocm/graph.hpp:27 enum Objective */
#define OCM_MINIMIZE 0
#define OCM_MAXIMIZE 1
/* include/ocm/solve.hpp:30 enum SccStrategy */
#define OCM_SCC_TARJAN 0
#define OCM_SCC_PARALLEL 1
#define OCM_SCC_OFF 2

typedef struct ocm_graph ocm_graph;
typedef struct ocm_session ocm_session;

/* include/ocm/solve.hpp:36 SolveOptions. engine schedule/workers/seed of the
 * reference's CPU engine have no meaning on the device and are not present. */
typedef struct {
    int32_t algo;      /* OCM_ALGO_*; HOWARD and HOWARD_PAR both run the device lane */
    int32_t objective; /* OCM_MINIMIZE / OCM_MAXIMIZE */
    int32_t scc;       /* OCM_SCC_*; TARJAN and PARALLEL both decompose into regions */
    int32_t device;    /* CUDA device ordinal */
    double epsilon;    /* accepted for signature parity (Lawler only), unused */
} ocm_solve_options;

/* include/ocm/solve.hpp:45 SolveStats + :54 Solution. The optimal cycle's
 * vertex list is returned through the cycle_buf argument of ocm_solve. */
typedef struct {
    int32_t has_cycle;
    int32_t exact;          /* mu_num/mu_den authoritative (integer weights) */
    int64_t mu_num;
    int64_t mu_den;         /* > 0, gcd(|num|, den) == 1 */
    double mu;
    uint32_t cycle_len;     /* full length (may exceed cycle_cap) */
    uint32_t outer_iters;   /* host iterations that rebuilt a policy */
    uint32_t spf_passes;    /* improvement passes incl. the final quiet one */
    uint32_t regions;
    uint32_t trivial_regions;
    uint32_t n_solved;      /* vertices in non-trivial regions */
    uint64_t m_solved;      /* intra-region edges streamed per improvement pass */
    uint64_t launches;      /* device kernel launches */
    uint64_t fixpoint_iters;/* pointer-jumping rounds + attach layers */
    double device_ms;       /* CUDA-event time of the device solve */
    double improve_ms;      /* CUDA-event time summed over improvement launches */
    double host_prep_ms;    /* host time of region split + upload (session create) */
    uint64_t h2d_bytes;     /* host->device bytes moved by the call (upload at create) */
    uint64_t d2h_bytes;     /* device->host bytes moved by this solve (flags + results) */
} ocm_solution;

const char* ocm_last_error(void);
int ocm_last_error_line(void);
const char* ocm_version(void);
int ocm_device_count(void);

int ocm_build_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                    const double* w, ocm_graph** out);
int ocm_parse_graph_text(const char* text, size_t len, const char* source, ocm_graph** out);
int ocm_read_graph_file(const char* path, ocm_graph** out);
/* Synthetic uniform digraph: every vertex has exactly deg out-edges, targets
 * and integer weights in [wlo, whi] drawn from a seeded counter hash. */
int ocm_generate_uniform(uint32_t n, uint32_t deg, int32_t wlo, int32_t whi, uint64_t seed,
                         ocm_graph** out);
/* Synthetic benchmark graphs (BASELINE.json configs). The same description
 * generates a host graph (ocm_generate, for checkers and small sizes) or a
 * session whose CSR is written directly into HBM (ocm_session_create_generated,
 * no host copy); both produce bit-identical graphs. */
#define OCM_GEN_UNIFORM 0  /* every vertex has exactly deg out-edges */
#define OCM_GEN_POWERLAW 1 /* deg(v) = min(dmax, floor(deg / sqrt(u_v))), tail exponent 3 */
#define OCM_GEN_POWERLAW_HUBS 2 /* out-degrees as OCM_GEN_POWERLAW; targets floor(n*u^2) scattered
                                   by a bijection: in-degree tail exponent 3 too (hub vertices) */
#define OCM_GEN_POWERLAW_WEB 3  /* as OCM_GEN_POWERLAW_HUBS with targets floor(n*u^8): in-degree
                                   density exponent ~2.14 (web graphs) */
typedef struct {
    int32_t kind;    /* OCM_GEN_* */
    uint32_t n;
    uint32_t deg;    /* uniform: out-degree; power-law: minimum out-degree */
    uint32_t dmax;   /* power-law: degree cap */
    int32_t wlo;     /* integer weights uniform in [wlo, whi] */
    int32_t whi;
    uint64_t seed;
} ocm_generator;
int ocm_generate(const ocm_generator* spec, ocm_graph** out);

/* include/ocm/model_gen.hpp:31 Scenario::Transition */
typedef struct {
    uint32_t from;
    uint32_t to;
    int64_t cost;
    int32_t acquires; /* enabled only while the server is free */
    int32_t releases; /* enabled only for the current holder */
} ocm_transition;
/* include/ocm/model_gen.hpp:67 generate_model(scenario, clients): the
 * reachable composite state space of `clients` interleaved copies of the
 * scenario, vertices in breadth-first discovery order. max_states bounds the
 * exploration (0 = the reference's kMaxModelStates, 5,000,000); exceeding it
 * returns OCM_E_LOGIC ("state space exceeds N states", std::length_error). */
int ocm_generate_model(uint32_t states, const ocm_transition* transitions, uint32_t n_transitions,
                       int32_t uses_server, uint32_t clients, uint64_t max_states,
                       ocm_graph** out);
void ocm_graph_free(ocm_graph* g);
uint32_t ocm_graph_n(const ocm_graph* g);
uint64_t ocm_graph_m(const ocm_graph* g);
int ocm_graph_integer_exact(const ocm_graph* g);
int ocm_graph_edges(const ocm_graph* g, uint32_t* src, uint32_t* dst, double* w);
/* The graph's forward CSR in place (graph.hpp:38-41: fwd_index n+1 offsets,
 * here 64-bit; fwd_target / fwd_weight m entries): read-only pointers owned
 * by the graph, valid until ocm_graph_free. */
int ocm_graph_csr(const ocm_graph* g, const uint64_t** fwd_index, const uint32_t** fwd_target,
                  const double** fwd_weight);

/* One-call front door (create session, solve, free). */
int ocm_solve(const ocm_graph* g, const ocm_solve_options* opt, ocm_solution* out,
              uint32_t* cycle_buf, uint32_t cycle_cap);

/* ocm::solve (solve.hpp:64) on the reference's own graph representation,
 * without building an ocm_graph: the forward CSR of ocm::Graph exactly as it
 * lies in the caller's memory (graph.hpp:38-41: fwd_index has n+1 EdgeId =
 * uint32 offsets, fwd_target m vertices, fwd_weight m doubles; edge id =
 * CSR position). The arrays are only read: pageable memory is staged through
 * the library's pinned ring, page-locked memory is copied directly. The
 * device checks them as build_graph would (graph.cpp:29-36: OCM_E_INVALID
 * "edge <e> endpoint out of range" / "edge <e> has non-finite weight", and
 * offsets that do not run from 0 to m) and derives integer_exact itself. */
int ocm_solve_csr(uint32_t n, uint32_t m, const uint32_t* fwd_index, const uint32_t* fwd_target,
                  const double* fwd_weight, const ocm_solve_options* opt, ocm_solution* out,
                  uint32_t* cycle_buf, uint32_t cycle_cap);
/* A resident session on the reference's CSR arrays (as ocm_solve_csr; the
 * arrays are only read during the call): repeated solves reuse the prepared
 * graph in HBM (ocm_session_solve / _values / _certify / _free). */
int ocm_session_create_csr(uint32_t n, uint32_t m, const uint32_t* fwd_index,
                           const uint32_t* fwd_target, const double* fwd_weight,
                           const ocm_solve_options* opt, ocm_session** out);

/* Resident sessions: create uploads the region-compacted CSR into HBM once;
 * each solve re-runs policy iteration from the initial policy on the device. */
int ocm_session_create(const ocm_graph* g, const ocm_solve_options* opt, ocm_session** out);
int ocm_session_solve(ocm_session* s, ocm_solution* out, uint32_t* cycle_buf, uint32_t cycle_cap);
/* Final per-vertex values of the last solve (original vertex order), the
 * plane written by the last value propagation: exact graphs give
 * value(v) = key_num[v] / lam_den[v] as a rational (key_num = wsum*den -
 * steps*num of the reference's (wsum, steps) pair); float graphs fill fval.
 * Vertices of trivial regions report 0. Any pointer may be NULL. */
int ocm_session_values(ocm_session* s, int64_t* key_num, int64_t* lam_num, int64_t* lam_den,
                       double* fval, uint32_t* succ_vertex);
/* Optimality certificate of the last solve, checked on the device in O(N+M)
 * over the solved (region-compacted) graph -- the size-independent parity
 * property at sizes the CPU oracle cannot reach (exact lane only):
 *   every intra-region edge v->t satisfies K[v] <= K[t] + w*den - num
 *   (K = value*den, lambda = num/den of v's region), the policy edge of every
 *   vertex attains K[v], and every region's anchor cycle is closed, anchored
 *   at its least vertex and of mean exactly lambda -- which together prove
 *   lambda is the region's minimum cycle mean. Counts are of violations. */
typedef struct ocm_certificate {
    uint64_t vertices, edges, regions; /* checked */
    uint64_t key_violations;           /* edges with K[v] > K[t] + w*den - num */
    uint64_t policy_violations;        /* policy edge missing or not attaining K[v] */
    uint64_t cycle_violations;         /* regions whose anchor cycle fails */
} ocm_certificate;
/* Exact value keys at full width (either exact lane): key = key_hi * 2^64 +
 * key_lo as a 128-bit two's complement, value = key / lam_den. The wide lane
 * (128-bit keys) runs when a weight needs more than 32 bits or a key could
 * leave +-2^62; ocm_session_values then returns OCM_E_RANGE for keys beyond
 * 64 bits. ocm_session_is_wide reports the lane of the session's last solve. */
/* Lambda of the (single) non-trivial region after each policy iteration of
 * the last solve -- the reference's HowardTrace (howard_par.hpp:588, which
 * records it when there is one region): exact lanes fill num/den, the float
 * lane f; *len = the number of iterations (at most 4096 entries kept). */
int ocm_session_lambda_trace(ocm_session* s, int64_t* num, int64_t* den, double* f, uint32_t cap,
                             uint32_t* len);
/* Debug trace of a session created with the environment variable
 * OCM_TRACE_ITERS=k (one rank): the policy edge ids and value keys (exact,
 * low 64 bits; float values in fval) after iteration `iter` < k of the last
 * solve -- what HowardTrace records per iteration (howard_par.hpp:588). */
int ocm_session_iter_trace(ocm_session* s, uint32_t iter, uint32_t* succ_edge, int64_t* key,
                           double* fval);
int ocm_session_keys_wide(ocm_session* s, int64_t* key_hi, uint64_t* key_lo);
int ocm_session_is_wide(const ocm_session* s);
int ocm_session_certify(ocm_session* s, ocm_certificate* out);
/* A session over a generated graph built in HBM (no host graph). */
int ocm_session_create_generated(const ocm_generator* spec, const ocm_solve_options* opt,
                                 ocm_session** out);
/* ---- sharded lane: vertices 1-D partitioned over `world`
 * ranks (one process per GPU). Every rank holds the prepared graph; rank r
 * improves the policy of vertices [r*chunk, (r+1)*chunk) only, and after
 * each improvement pass the ranks exchange the policy slices (all-gather of
 * succ_e, succ_v, succ_w in chunk-sized pieces) and max-reduce the per-region
 * change flags (changed0/changed1, `regions` int32 each); cycle detection and
 * value determination then run replicated. Pass exactly one of g / spec. */
typedef struct {
    uint32_t rank, world, chunk;
    uint32_t own_lo, own_hi, n;
    void* succ_e;          /* uint32[world*chunk] */
    void* succ_v;          /* uint32[world*chunk] */
    void* succ_w;          /* int32 (exact) or double (float) [world*chunk] */
    uint32_t succ_w_bytes; /* 4 or 8 */
    uint32_t regions;      /* entries of changed0/changed1 */
    void* changed0;        /* int32[regions] */
    void* changed1;
    void* stream;          /* cudaStream_t the session launches on */
} ocm_shard_buffers;
int ocm_session_create_shard(const ocm_graph* g, const ocm_generator* spec,
                             const ocm_solve_options* opt, uint32_t rank, uint32_t world,
                             ocm_session** out);
int ocm_session_shard_buffers(ocm_session* s, ocm_shard_buffers* out);
/* One launch up to the next exchange point; *done = 1 when the solve finished
 * (then read it with ocm_session_shard_finish). The first call of a solve
 * starts it from the initial policy. */
int ocm_session_shard_step(ocm_session* s, int32_t* done);
int ocm_session_shard_finish(ocm_session* s, ocm_solution* out, uint32_t* cycle_buf,
                             uint32_t cycle_cap);
/* ---- fused sharded lane: one persistent launch per solve per rank. During
 * the improvement pass every changed policy entry is stored straight into
 * the peers' replicas (NVLink stores into peer memory) and two cross-rank
 * barriers per iteration (system-scope atomics on the peers' barrier words)
 * replace the host exchange. Each rank publishes its buffer descriptor, all
 * ranks connect with the full rank-ordered list (use_ipc = 1 across
 * processes: the handles are opened with cudaIpcOpenMemHandle; 0 within one
 * process: raw device pointers, peer access enabled when the devices
 * differ), then every rank launches and finishes. All ranks must launch:
 * a missing peer ends the solve with an error after a bounded wait. */
typedef struct {
    uint64_t ptr[6];           /* succ_e, succ_v, succ_w, changed0, changed1, barrier word */
    unsigned char ipc[6][64];  /* cudaIpcMemHandle_t of each */
    int32_t device;
    uint32_t rank;
} ocm_shard_peer;
int ocm_session_shard_peer_info(ocm_session* s, ocm_shard_peer* out);
int ocm_session_shard_connect(ocm_session* s, const ocm_shard_peer* peers, uint32_t world,
                              int32_t use_ipc);
int ocm_session_shard_fused_launch(ocm_session* s);
int ocm_session_shard_fused_finish(ocm_session* s, ocm_solution* out, uint32_t* cycle_buf,
                                   uint32_t cycle_cap);
/* Vertex count of the session's graph. */
uint32_t ocm_session_n(const ocm_session* s);
/* The CUDA stream the session launches on (cudaStream_t). */
void* ocm_session_stream(ocm_session* s);
void ocm_session_free(ocm_session* s);

#ifdef __cplusplus
}
#endif
#endif /* OCM_B200_H */
