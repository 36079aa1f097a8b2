/*
 * pmx_b200.h — C ABI of the B200 backend for the accelerated-expression hot
 * path of the PMExpr reference runtime (arXiv 2211.00621, reference package
 * `pmx`, paths below are relative to /root/reference/pkg/src).
 *
 * The reference has no FFI: its hot path is a set of module-level Python
 * functions in pmx/interp.py that a host binding can replace by assignment.
 * Each entry point here replaces one of them (file:line of the function it
 * stands in for is given on each declaration); the Python package
 * `paper_2211_00621_b200` binds them through ctypes.
 *
 * Conventions
 *  - Every data pointer is a DEVICE pointer owned by the caller. The library
 *    never allocates device memory behind the caller's back; operations that
 *    need scratch take a caller-provided workspace (query its size first).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *    asynchronous on that stream, re-entrant, and thread-safe across streams.
 *  - Return value: 0 = launched, <0 = argument / CUDA error (message in
 *    pmx_last_error(), thread-local). User-level runtime errors (division by
 *    zero, log domain, out-of-bounds, ...) are detected ON THE DEVICE and
 *    recorded in a 64-bit error word `err` (device pointer, nullable):
 *        err == PMX_ERR_NONE            no error
 *        err  = (index << 8) | code     first failing element in element order
 *    The word is combined with atomicMin, so the reported element is the
 *    smallest failing index — the same element the reference reports, whose
 *    workers re-raise in chunk order (pmx/interp.py:291) and whose chunks are
 *    contiguous and ascending (pmx/interp.py:273-276).
 *    Codes are enum pmx_code; messages match pmx/interp.py:379-436.
 */
#ifndef PMX_B200_H
#define PMX_B200_H

#include <stdint.h>
#include <stddef.h>

#if defined(__GNUC__)
#define PMX_API __attribute__((visibility("default")))
#else
#define PMX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PMX_ABI_VERSION 1
#define PMX_ERR_NONE 0xFFFFFFFFFFFFFFFFull

/* ---- element types: PMExpr Int = int64, Float = fp64;
 *      f32 / i32 are storage-only narrowings used by the benchmark configs. */
enum pmx_dtype {
    PMX_F32 = 0,
    PMX_F64 = 1,
    PMX_I64 = 2,
    PMX_I32 = 3,
    PMX_BOOL = 4   /* stored as uint8 */
};

/* ---- device-detected runtime errors (pmx/interp.py:379-436, 151-154) */
enum pmx_code {
    PMX_OK = 0,
    PMX_E_DIVI0 = 1,       /* "integer division by zero"          interp.py:387-388 */
    PMX_E_MODI0 = 2,       /* "integer modulo by zero"            interp.py:392-393 */
    PMX_E_DIVF0 = 3,       /* "float division by zero"            interp.py:407-408 */
    PMX_E_LOG_DOMAIN = 4,  /* "log: math domain error"            interp.py:428-432 */
    PMX_E_EXP_RANGE = 5,   /* "exp: math range error"             interp.py:428-432 */
    PMX_E_SQRT_NEG = 6,    /* "sqrtf of a negative number"        interp.py:433-436 */
    PMX_E_OOB = 7,         /* "get index i out of bounds ..."     interp.py:536-541 */
    PMX_E_TENSOR_OOB = 8,  /* "tensor index k out of bounds ..."  runtime.py:69-73 */
    PMX_E_NEVER = 9,       /* "reached a never expression"        interp.py:133-135 */
    PMX_E_F32_RANGE = 10,  /* result not representable in the f32 storage type */
    PMX_E_SIN_COS_INF = 11,/* "sin/cos: math domain error" (inf argument)      */
    PMX_E_PEER_TIMEOUT = 12,/* a peer GPU did not deliver its partial (20 s)   */
    PMX_E_RECURSION = 13   /* linear recursion run as a loop exceeded its bound   */
};

/* ---- scalar-function bytecode ------------------------------------------
 * A PMExpr lambda restricted to scalar code (the bodies the well-formedness
 * rules admit on the functional backend, pmx/wellformed.py:32-53) is compiled
 * by the host into a register program. Registers are untyped 64-bit; each op
 * fixes the interpretation (int64 or fp64, i.e. the reference's value types).
 * Operand byte: 0..31 register, 32..63 constant-pool slot (value - 32).
 * Inputs: map f -> r0 = x[j], r1 = j; map2 -> r0 = x, r1 = y, r2 = j;
 *         reduce/fold op -> r0 = acc, r1 = x; loop body -> r0 = i.       */
#define PMX_MAX_INSNS 96
#define PMX_MAX_CONSTS 32
#define PMX_MAX_REGS 32
#define PMX_MAX_ARRAYS 6
#define PMX_MAX_RANK 4

enum pmx_op {
    PMX_OP_NOP = 0, PMX_OP_MOV,
    PMX_OP_ADDI, PMX_OP_SUBI, PMX_OP_MULI, PMX_OP_DIVI, PMX_OP_MODI, PMX_OP_NEGI,
    PMX_OP_ADDF, PMX_OP_SUBF, PMX_OP_MULF, PMX_OP_DIVF, PMX_OP_NEGF,
    PMX_OP_EQI, PMX_OP_NEQI, PMX_OP_LTI, PMX_OP_GTI, PMX_OP_LEQI, PMX_OP_GEQI,
    PMX_OP_EQF, PMX_OP_LTF, PMX_OP_GTF, PMX_OP_LEQF, PMX_OP_GEQF,
    PMX_OP_INT2FLOAT, PMX_OP_FLOOR,
    PMX_OP_EXP, PMX_OP_LOG, PMX_OP_SIN, PMX_OP_COS, PMX_OP_SQRT,
    PMX_OP_NOT, PMX_OP_SELECT,      /* dst = a ? b : c                        */
    PMX_OP_GET,                     /* dst = arrays[c][a]  (bounds-checked)   */
    PMX_OP_LEN,                     /* dst = len(arrays[c])                   */
    PMX_OP_TGET,                    /* dst = tensor[c][r_a .. r_a+rank)       */
    PMX_OP_TSET,                    /* tensor[c][r_a ..] = r_b ; dst ignored  */
    PMX_OP_NEVER,                   /* raise PMX_E_NEVER                      */
    PMX_OP_EQB,                     /* bool equality (match on Bool literal)  */
    PMX_OP_JZ,                      /* if r_a == 0: pc = b | c << 8 (match)   */
    PMX_OP_JMP,                     /* pc = b | c << 8                        */
    PMX_OP_FAIL,                    /* raise error code b (enum pmx_code)     */
    PMX_OP_COUNT
};

typedef struct pmx_insn {
    uint8_t op, dst, a, b, c, pad0, pad1, pad2;
} pmx_insn;

/* A captured sequence (for GET/LEN) or tensor view (for TGET/TSET). */
typedef struct pmx_array {
    void* data;             /* device pointer to the ROOT buffer (Alg. 2 root) */
    int64_t offset;         /* element offset of the view inside the root      */
    int64_t shape[PMX_MAX_RANK];
    int32_t rank;           /* 1 for sequences                                 */
    int32_t dtype;          /* enum pmx_dtype                                  */
} pmx_array;

typedef struct pmx_program {
    int32_t n_insns;
    int32_t n_inputs;
    int32_t out;            /* operand holding the result                      */
    int32_t out_is_float;   /* 1 if the result register holds an fp64          */
    int32_t n_arrays;
    int32_t pad;
    pmx_insn insns[PMX_MAX_INSNS];
    int64_t consts[PMX_MAX_CONSTS];     /* bit patterns (int64 or fp64)        */
    pmx_array arrays[PMX_MAX_ARRAYS];
} pmx_program;

/* ---- library ------------------------------------------------------------ */
PMX_API int         pmx_abi_version(void);
PMX_API const char* pmx_last_error(void);
/* Recognised fast-path kind of a program (for tests/diagnostics): 0 = VM. */
PMX_API int         pmx_program_kind(const pmx_program* f, int32_t role);
/* Reset an error word to PMX_ERR_NONE on `stream`. */
PMX_API int         pmx_err_reset(uint64_t* err, void* stream);

/* ---- skeletons ------------------------------------------------------------ */

/* y[j] = f(x[j]) for j in [0,n).           replaces eval_map   interp.py:294-304 */
PMX_API int pmx_map(const pmx_program* f, const void* x, int32_t x_dtype,
            void* y, int32_t y_dtype, int64_t n, uint64_t* err, void* stream);

/* z[j] = f(x[j], y[j]).                    replaces eval_map2  interp.py:307-319
 * (the length check of interp.py:151-154 is done by the caller: both inputs
 * have length n by construction of the call).                                  */
PMX_API int pmx_map2(const pmx_program* f, const void* x, int32_t x_dtype,
             const void* y, int32_t y_dtype, void* z, int32_t z_dtype,
             int64_t n, uint64_t* err, void* stream);

/* Workspace for pmx_map_reduce / pmx_fold over n elements. It must be zeroed
 * before first use; every call leaves it zeroed again (the completion ticket
 * is reset by the last CTA), so one workspace serves a whole stream.        */
PMX_API size_t pmx_reduce_workspace_bytes(int64_t n);

/* out = fold(op, init, map(f, x)) evaluated as a deterministic parallel tree:
 * per-thread partials, warp shuffle, shared-memory block combine, then the
 * last CTA to finish folds the per-CTA partials in CTA order. `init` is
 * applied exactly once (debug-mode semantics, interp.py:329-330; the parallel
 * reference folds it into every chunk, interp.py:332-333, which is only
 * equivalent for a neutral `init`).
 * f == NULL means identity (plain reduce).  y (nullable) materialises map(f,x).
 * Float sums/products accumulate in fp64 (the reference's Float), whatever the
 * storage dtype; `init` and `out` are in acc_dtype (PMX_F64 or PMX_I64).
 *                                     replaces eval_reduce interp.py:328-343
 *                                              + _fold      interp.py:322-325 */
PMX_API int pmx_map_reduce(const pmx_program* f, const pmx_program* op,
                   const void* x, int32_t x_dtype, int64_t n,
                   const void* init_host, int32_t acc_dtype, void* out,
                   void* y, int32_t y_dtype,
                   void* workspace, size_t workspace_bytes,
                   uint64_t* err, void* stream);

/* Left fold on the device: out = foldl op init x.  Runs on one thread in
 * element order, except for operators whose result is independent of the
 * bracketing (int add/mul/min/max, float min/max), which use the parallel
 * tree when a workspace (nullable) is given.
 *                                     replaces foldl builtin interp.py:461-463 */
PMX_API int pmx_fold(const pmx_program* op, const void* x, int32_t x_dtype, int64_t n,
             const void* init_host, int32_t acc_dtype, void* out,
             void* workspace, size_t workspace_bytes,
             uint64_t* err, void* stream);

/* Row functions: out[r] = fold over row r of x (rows delimited by int64
 * offsets[nrows+1]) — `map (lam row. reduce op acc (map g row)) rows`,
 * `foldl op acc row` and `reduce op acc row` (g == NULL).  Inside a map body
 * the reference runs these sequentially (interp.py:82-84): a left fold from
 * init in element order.  g: r0 = x, r1 = index in the row; op: r0 = acc,
 * r1 = value.  out has out_dtype; errors report the row index.
 *                                     replaces eval_map over [[a]] with a row
 *                                     function, interp.py:294-304 + 322-343 */
PMX_API int pmx_map_rows_fold(const pmx_program* g, const pmx_program* op, const void* x, int32_t x_dtype,
                      const int64_t* offsets, int64_t nrows, const void* init_host, void* out,
                      int32_t out_dtype, uint64_t* err, void* stream);

/* Parallel loop: body(i) for i in [0,n), effects through TSET on the tensor
 * views in body->arrays (already rebased into their device roots by the
 * host's marshal_in, Alg. 2).           replaces eval_loop interp.py:346-358 */
PMX_API int pmx_loop(const pmx_program* body, int64_t n, uint64_t* err, void* stream);

/* seqLoop: persistent on-device iteration of a parallel step.
 * state has m elements (fp64), scratch m + 8 (the tail holds the grid-barrier
 * word of the specialised kernel); for t in [0,steps):
 *     state'[j] = f(state[j], j, t)   where f may GET from the previous state
 *                                     through arrays[0] (set by the library).
 * One launch, grid-wide barrier between steps.   (recursion used as a
 * sequential device loop: programs/rk4.pmx:38-40, programs/viterbi.pmx:35-48) */
PMX_API int pmx_seq_loop(const pmx_program* f, double* state, double* scratch,
                 int64_t m, int64_t steps, uint64_t* err, void* stream);

/* The same with the initial state read from `init` (left unchanged) and the
 * result in `state`: the copy of a caller's sequence into the iteration
 * buffers is fused into step 0.       (seqLoop's input is an immutable value) */
PMX_API int pmx_seq_loop_from(const pmx_program* f, const double* init, double* state, double* scratch,
                      int64_t m, int64_t steps, uint64_t* err, void* stream);

/* offsets[0]=0, offsets[i+1] = offsets[i] + lengths[i]  (int64).  Used to
 * flatten an irregular sequence: flatten is then the values buffer itself.
 *                                     replaces FlattenE interp.py:161-166 */
PMX_API int pmx_scan_lengths(const int64_t* lengths, int64_t* offsets, int64_t n,
                     void* stream);

/* offsets[i] = i * row_len for i in [0, nrows]: the row offsets of a regular
 * nested sequence, so row kernels take one layout for regular and irregular
 * rows.                              used by the row-fold map (interp.py:294-304) */
PMX_API int pmx_row_offsets(int64_t* offsets, int64_t nrows, int64_t row_len, void* stream);

/* ---- run-time kernel specialisation ---------------------------------------
 * A lambda the library does not recognise runs, above a size threshold, in
 * the streaming skeleton kernel specialised to it: its bytecode is translated
 * to C++ with the same semantics and compiled by NVRTC for sm_100a (cached per
 * program shape; constants and captured arrays stay kernel arguments). Below
 * the threshold (or with mode 0) it runs in the bytecode interpreter.
 * mode: 0 = interpreter only, 1 = always specialise, 2 = auto (default; the
 * PMX_JIT environment variable sets the initial mode). Returns the old mode. */
PMX_API int pmx_jit_set_mode(int32_t mode);
/* Kernels compiled / launched through the specialised path so far.          */
PMX_API int pmx_jit_stats(int64_t* compiled, int64_t* launched);
/* The generated element functor for skeleton kind 0 = map, 1 = map2,
 * 2 = loop body (diagnostics); returns its length or < 0.                   */
PMX_API int pmx_jit_source(const pmx_program* f, int32_t kind, char* buf, size_t len);
/* Generate and compile (no GPU needed, nothing loaded) the kernel for kind
 * with element dtypes x, y (map2: z = result dtype); 0 = compiles.          */
PMX_API int pmx_jit_compile_check(const pmx_program* f, int32_t kind, int32_t x_dtype,
                                  int32_t y_dtype, int32_t z_dtype);

/* ---- multi-GPU reduce: partials combined over NVLink peer memory ----------
 * One process per GPU. Each rank creates a mailbox (pmx_peer_mailbox_create,
 * zeroed, 512 B), exports its IPC handle, receives every peer's handle through
 * the host's process group and maps them (pmx_peer_open). A pmx_peer_group
 * then holds every rank's mailbox pointer (own pointer at [rank]).
 * pmx_map_reduce_peers is pmx_map_reduce over this rank's shard whose last CTA
 * also exchanges the shard partials through the mailboxes and folds the
 * contributing ones in rank order: `out` is the global result on every rank,
 * from one kernel and no collective call. Each rank's shard folds from its
 * init; partials fold left in rank order (interp.py:334-336); empty shards are
 * dropped (interp.py:276) except rank 0's, which always contributes its init.
 * The host layer (shard.py) passes acc as rank 0's init and the operator's
 * identity on the other ranks, so acc is applied once, as on one GPU.
 * `epoch` must be incremented (from 1) by every rank before each call; all
 * ranks must make the same sequence of calls.       replaces eval_reduce's
 * chunk combine across GPUs (interp.py:334-336) / an NCCL all-gather + fold. */
#define PMX_MAX_PEERS 16
#define PMX_IPC_HANDLE_BYTES 64
typedef struct pmx_peer_group {
    int32_t rank;
    int32_t world;                       /* <= PMX_MAX_PEERS                  */
    uint64_t epoch;                      /* >= 1, +1 per call                 */
    uint64_t* mbox[PMX_MAX_PEERS];       /* device pointers, [rank] = own     */
} pmx_peer_group;

PMX_API int pmx_peer_mailbox_create(void** mbox_out, void* ipc_handle_out /* 64 B */);
PMX_API int pmx_peer_mailbox_destroy(void* mbox);
PMX_API int pmx_peer_open(const void* ipc_handle /* 64 B */, void** mbox_out);
PMX_API int pmx_peer_close(void* mbox);
PMX_API int pmx_map_reduce_peers(const pmx_program* f, const pmx_program* op,
                   const void* x, int32_t x_dtype, int64_t n,
                   const void* init_host, int32_t acc_dtype, void* out,
                   void* workspace, size_t workspace_bytes,
                   const pmx_peer_group* group, uint64_t* err, void* stream);

/* ---- case-study kernels ---------------------------------------------------- */

/* RK4 sweep of programs/rk4.pmx:11-45: out[k*4 + c] = integrate(p[k], init, steps)
 * fp64, evaluation order of the program (no contraction).                     */
PMX_API int pmx_rk4_sweep_f64(const double* params, int64_t n, const double* init4,
                      int32_t steps, double h, double* out, void* stream);

/* The paper's ODE study output: the same sweep, also
 * recording state component `comp` (0..3) after every step into the N x M
 * tensor trace[k * steps + m] (row-major, device pointer: a tensor view's
 * root + offset).  out[k*4 + c] receives the final states.                   */
PMX_API int pmx_rk4_trace_f64(const double* params, int64_t n, const double* init4, int32_t steps,
                      double h, int32_t comp, double* trace, double* out, void* stream);

/* Log-space HMM forward for nsig signals of length T:
 * out_ll[s] = log P(obs[s, 0:T]).  log_pi[S], A[S*S] row-major probabilities
 * (A[i*S+j] = P(j | i)), log_E[S*K] (log_E[j*K+k]), obs int32 [nsig*T].
 * Computed as a scaled linear-space recursion in fp32 with an fp64 running
 * log-scale per signal.                                                        */
PMX_API size_t pmx_hmm_forward_workspace_bytes(int32_t S, int64_t nsig);
PMX_API int pmx_hmm_forward_f32(const float* log_pi, const float* A, const float* log_E,
                        int32_t S, int32_t K, const int32_t* obs, int64_t nsig,
                        int32_t T, double* out_ll, void* workspace,
                        size_t workspace_bytes, void* stream);
/* S = 1024 runs on the tensor cores with fp16 operands (exact power-of-two
 * scalings of A, u and each symbol's emission column).  A range guard flags
 * every signal whose per-step predicted emission mass falls below 2^-8 (where
 * fp16's subnormal range could cost more than the 1e-5 budget); flagged
 * signals are recomputed by the TF32 kernel in the same call, decided on the
 * device.  This returns how many signals the last call on `workspace` re-ran
 * (synchronises `stream`; -1 on a CUDA error).                               */
PMX_API int64_t pmx_hmm_forward_rerun_count(const void* workspace, int32_t S, int64_t nsig, void* stream);

/* Viterbi (programs/viterbi.pmx:23-59) for nsig signals: path[s*T + t] and
 * logp[s]; ties resolve to the smallest state index (strict > in argmax,
 * viterbi.pmx:142-145).  log_A[S*S], log_E[S*K], log_pi[S] in fp64.           */
PMX_API size_t pmx_viterbi_workspace_bytes(int32_t S, int64_t nsig, int32_t T);
PMX_API int pmx_viterbi_f64(const double* log_pi, const double* log_A,
                    const double* log_E, int32_t S, int32_t K,
                    const int32_t* obs, int64_t nsig, int32_t T,
                    int32_t* path, double* logp, void* workspace,
                    size_t workspace_bytes, void* stream);
/* Max-plus cells (candidate (i, j) pairs per signal-step) the last
 * pmx_viterbi_f64 call on `workspace` evaluated in the pruned (branch and
 * bound) kernel, S in {256, 512, 1024}: the roofline's work count.
 * Synchronises `stream`; -1 on a CUDA error.                                */
PMX_API int64_t pmx_viterbi_visited_cells(const void* workspace, int32_t S, int64_t nsig, int32_t T,
                                  void* stream);

/* Softmax regression (programs/nn.pmx:22-49): mean cross-entropy loss and its
 * analytic gradients for npts points, one fused launch.  x [npts*nin] fp64,
 * y [npts] int32 class labels, w [nin*nout], b [nout]; outputs loss [1],
 * dw [nin*nout], db [nout] (device pointers).  nin <= 64, nout <= 32.
 * Runtime errors (class label out of range, exp overflow, npts == 0 ->
 * "float division by zero" as divf _ 0.0) go to the error word.            */
PMX_API size_t pmx_nn_workspace_bytes(int64_t npts, int32_t nin, int32_t nout);
PMX_API int pmx_nn_softmax_grad_f64(const double* x, const int32_t* y, const double* w, const double* b,
                            int64_t npts, int32_t nin, int32_t nout, double* loss, double* dw,
                            double* db, void* workspace, size_t workspace_bytes, uint64_t* err,
                            void* stream);

/* k-NN classification: label of each query = majority
 * vote of the k nearest train points by squared L2 distance, ties by smaller
 * train index, vote ties to the smaller label.  train [ntr*d] f32, query
 * [nq*d] f32, labels int32 in [0,ncls).  out_idx (nullable) [nq*k].          */
PMX_API size_t pmx_knn_workspace_bytes(int64_t ntr, int64_t nq, int32_t d, int32_t k);
PMX_API int pmx_knn_f32(const float* train, const int32_t* labels, int64_t ntr,
                const float* query, int64_t nq, int32_t d, int32_t k,
                int32_t ncls, int32_t* out_label, int32_t* out_idx,
                void* workspace, size_t workspace_bytes, void* stream);

/* k-mer (de Bruijn) HMM forward, S = 4^kmer states; predecessors of j are j
 * (stay, p_stay) and (j >> 2) | (b << (2*kmer-2)) for b in 0..3 (p_step each).
 * log_E[S*K], obs int32 [nsig*T]; out_ll[s] fp64.  Uniform initial state.    */
PMX_API size_t pmx_hmm_kmer_workspace_bytes(int32_t kmer, int64_t nsig);
PMX_API int pmx_hmm_kmer_forward_f32(int32_t kmer, float p_stay, float p_step,
                             const float* log_E, int32_t K,
                             const int32_t* obs, int64_t nsig, int32_t T,
                             double* out_ll, void* workspace,
                             size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PMX_B200_H */
