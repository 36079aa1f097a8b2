// Internal interface between the skeleton launchers (skeletons.cu) and the
// run-time kernel compiler (jit.cu). Not part of the C ABI.
#pragma once
#include "common.cuh"

namespace pmx {

static const int kStreamThreads = 256;
static const int kReduceBlocksPerSM = 8;

// Fast-path kinds returned by pmx_program_kind (role 0 = unary map function
// r0 = x, role 1 = binary reduce operator r0 = acc, r1 = x).
enum FastKind {
    K_VM = 0,
    K_IDENTITY = 1,
    K_AFFINE_F = 2,   // y = a*x + b (fp64 semantics; flags choose mul/add)
    K_AFFINE_I = 3,   // y = a*x + b (int64 wrap)
    K_ADD_F = 10, K_MUL_F = 11, K_MIN_F = 12, K_MAX_F = 13,
    K_ADD_I = 20, K_MUL_I = 21, K_MIN_I = 22, K_MAX_I = 23,
};

int stream_grid(int64_t n, int cap);

// Run-time compiled (NVRTC) skeleton kernels specialised to one lambda.
// Each returns 0 when launched, 1 when the JIT declines (disabled for this
// size, or a construct it does not generate) so the caller runs the
// interpreter, <0 on error (pmx_last_error).
bool jit_wanted(int64_t n);
int jit_map(const pmx_program* f, const void* x, int xt, void* y, int yt, int64_t n,
            uint64_t* err, cudaStream_t st);
int jit_map2(const pmx_program* f, const void* x, int xt, const void* y, int yt, void* z, int zt,
             int64_t n, uint64_t* err, cudaStream_t st);
int jit_loop(const pmx_program* body, int64_t n, uint64_t* err, cudaStream_t st);
int jit_reduce_generic(const pmx_program* f, const pmx_program* op, const void* x, int xt, int64_t n,
                       const void* init_host, int acc_dtype, void* out, void* ws, cudaStream_t st, uint64_t* err);
int jit_seq_loop(const pmx_program* f, const double* src, double* a, double* b, int64_t m, int64_t steps, unsigned* bar,
                 uint64_t* err, cudaStream_t st);
int jit_map_reduce(const pmx_program* f, int okind, const void* x, int xt, int64_t n,
                   const void* init_host, void* out, void* y, int yt, void* ws, cudaStream_t st,
                   const pmx_peer_group* pg, uint64_t* err);

}  // namespace pmx
