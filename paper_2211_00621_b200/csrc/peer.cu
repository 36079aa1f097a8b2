// Host side of the peer-memory combine (peer.cuh): mailbox allocation and
// CUDA IPC export/import. A mailbox is 2 parities x PMX_MAX_PEERS slots x
// (value, flag) u64 = 512 B of device memory, zeroed at creation (flag epoch
// 0 never matches a launch, epochs start at 1).
#include <string.h>
#include "common.cuh"

using namespace pmx;

static_assert(sizeof(cudaIpcMemHandle_t) == PMX_IPC_HANDLE_BYTES, "IPC handle size");

extern "C" {

int pmx_peer_mailbox_create(void** mbox_out, void* handle_out) {
    PMX_REQUIRE(mbox_out && handle_out, "pmx_peer_mailbox_create: null argument");
    const size_t bytes = 2 * PMX_MAX_PEERS * 2 * sizeof(uint64_t);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        set_last_error("peer mailbox: %s", cudaGetErrorString(e));
        return -2;
    }
    memcpy(handle_out, &h, sizeof(h));
    *mbox_out = p;
    return 0;
}

int pmx_peer_mailbox_destroy(void* mbox) {
    if (!mbox) return 0;
    cudaError_t e = cudaFree(mbox);
    if (e != cudaSuccess) { set_last_error("peer mailbox free: %s", cudaGetErrorString(e)); return -2; }
    return 0;
}

int pmx_peer_open(const void* handle, void** mbox_out) {
    PMX_REQUIRE(handle && mbox_out, "pmx_peer_open: null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) { set_last_error("peer open: %s", cudaGetErrorString(e)); return -2; }
    *mbox_out = p;
    return 0;
}

int pmx_peer_close(void* mbox) {
    if (!mbox) return 0;
    cudaError_t e = cudaIpcCloseMemHandle(mbox);
    if (e != cudaSuccess) { set_last_error("peer close: %s", cudaGetErrorString(e)); return -2; }
    return 0;
}

}  // extern "C"
