/*
 * bitpipe_comm.h -- C ABI of the BitPipe runtime context (part of
 * libbitpipe_b200.so): the communicator, message-slot, event and CUDA-graph
 * entry points of SURVEY §8(b)'s "minimal C exports", for hosts that drive
 * the pipeline without torch.distributed (a C++ or FFI host).
 *
 * The reference has no FFI (pure-Python API); what these
 * replace is the SPEC's train-step plumbing:
 *   bp_init / bp_comm_split   -> the per-link and replica-pair groups of the
 *                                executor (runtime/distributed.py)
 *   bp_send / bp_recv         -> "activations/gradients flow along schedule
 *                                edges", one message =
 *                                message_size bytes (core.py:150-157)
 *   bp_allreduce_mean         -> the eager replica-pair gradient mean after a
 *                                stage's last backward
 *   bp_graph_*                -> CUDA-graph capture / replay of a step
 * The in-tree Python executor makes the same calls through torch.distributed
 * (NCCL) and torch.cuda.CUDAGraph; both paths use the same NCCL library
 * (resolved with dlopen("libnccl.so.2"), reusing the copy torch already
 * loaded).
 *
 * Conventions as in bitpipe.h: device pointers owned by the caller, streams
 * as void*, int status (BP_OK / BP_ERR_*) with bp_last_error().  NCCL
 * failures return BP_ERR_COMM with the NCCL error string.  A bp_ctx owns
 * its communicator and the slot slabs allocated through it; bp_destroy
 * frees both (never caller memory).
 */
#ifndef BITPIPE_B200_COMM_H
#define BITPIPE_B200_COMM_H

#include <stddef.h>
#include <stdint.h>

#include "bitpipe.h"

#ifdef __cplusplus
extern "C" {
#endif

#define BP_ERR_COMM 4
#define BP_NCCL_ID_BYTES 128

typedef struct bp_ctx bp_ctx;

/* 1 if an NCCL library is already loaded in the process (no loading, no
 * device work); 2 if none is loaded yet but libnccl.so.2 can be found (the
 * probe loads and unloads it); 0 if there is none.  The other communicator
 * calls load libnccl.so.2 on first use when none is loaded; that copy then
 * stays in the process and a later torch import reuses it (same soname), so
 * a host that also uses torch must import torch first. */
BP_API int bp_comm_available(void);
/* A fresh NCCL unique id (rank 0 creates it, the host broadcasts the 128
 * bytes to every rank out of band). */
BP_API int bp_nccl_unique_id(void* id_out);
/* One communicator over `world` ranks on CUDA `device` (collective: every
 * rank calls it with the same id). */
BP_API int bp_init(int rank, int world, const void* nccl_id, int device, bp_ctx** ctx_out);
/* Sub-communicator of the ranks passing the same `color`, ordered by `key`
 * (collective over ctx): directed P2P links, replica-pair stage groups.
 * color < 0: this rank joins none (*ctx_out = NULL). */
BP_API int bp_comm_split(bp_ctx* ctx, int color, int key, bp_ctx** ctx_out);
BP_API int bp_comm_rank(const bp_ctx* ctx);
BP_API int bp_comm_size(const bp_ctx* ctx);
/* Message slots: `count` device buffers of `bytes` each, one slab owned by
 * ctx (freed by bp_destroy); *base_out = first slot, slot i at base + i*bytes
 * rounded up to 256 B (bp_slot_stride). */
BP_API int bp_slots_alloc(bp_ctx* ctx, size_t bytes, int count, void** base_out);
BP_API size_t bp_slot_stride(size_t bytes);
/* Point-to-point messages (asynchronous on `stream`).  The receiver posts
 * its receives from a peer in the order the peer sends them. */
BP_API int bp_send(bp_ctx* ctx, int peer, const void* ptr, size_t bytes, void* stream);
BP_API int bp_recv(bp_ctx* ctx, int peer, void* ptr, size_t bytes, void* stream);
/* Bracket several bp_send / bp_recv into one fused NCCL group. */
BP_API int bp_group_start(void);
BP_API int bp_group_end(void);
/* In-place mean over the communicator's ranks of n elements (BP_F32 or
 * BP_BF16), asynchronous on `stream`. */
BP_API int bp_allreduce_mean(bp_ctx* ctx, void* ptr, size_t n, int dtype, void* stream);
/* Destroys the communicator and frees the ctx's slot slabs (sub-contexts
 * are destroyed separately). */
BP_API int bp_destroy(bp_ctx* ctx);

/* Events (cudaEventDisableTiming) for cross-stream ordering. */
BP_API int bp_event_create(void** ev_out);
BP_API int bp_event_record(void* ev, void* stream);
BP_API int bp_stream_wait_event(void* stream, void* ev);
BP_API int bp_event_destroy(void* ev);

/* CUDA-graph capture of everything issued on `stream` (and on streams that
 * join it through events) between begin and end; launch replays it. */
BP_API int bp_graph_begin(void* stream);
BP_API int bp_graph_end(void* stream, void** graph_exec_out);
BP_API int bp_graph_launch(void* graph_exec, void* stream);
BP_API int bp_graph_destroy(void* graph_exec);

/* ------------------------------------------------------ peer memory ----
 * The NCCL-free transport of the train step (runtime/peer.py): each rank
 * exports its message-slot slab, its flag mailbox and its stage gradient
 * buffers; a sender copies a message straight into the receiver's slot
 * (copy engine; NVLink when the receiver is another GPU) and raises the
 * slot's flag in the receiver's mailbox; the receiver's stream waits on the
 * flag.  The replica pair of a stage reads each other's gradient through
 * the imported pointer inside bp_adam (fused peer-read replica mean).
 * Replaces, like bp_send / bp_recv / bp_allreduce_mean above, the SPEC's
 * message passing and replica allreduce.
 */
#define BP_IPC_HANDLE_BYTES 64
/* Export the allocation containing device pointer `ptr`: 64 handle bytes
 * (cudaIpcMemHandle_t) and the byte offset of ptr inside it. */
BP_API int bp_ipc_export(const void* ptr, void* handle_out, size_t* offset_out);
/* Map a peer's exported allocation into this process (current device);
 * *base_out + offset addresses the peer's pointer.  Opening one handle
 * again returns the same mapping (reference counted). */
BP_API int bp_ipc_open(const void* handle, void** base_out);
BP_API int bp_ipc_close(void* base);
/* Asynchronous copy on `stream` between any two device pointers (local,
 * peer GPU or imported). */
BP_API int bp_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);
/* Stream-ordered 32-bit flags (no kernel, no host): set writes `value` to
 * `addr` after everything issued before it on `stream` (release); wait
 * blocks `stream` until (int32)(*addr - value) >= 0. */
BP_API int bp_flag_set(void* stream, void* addr, uint32_t value);
BP_API int bp_flag_wait(void* stream, const void* addr, uint32_t value);
/* Same wait as a one-thread polling kernel on `stream` (acquire loads,
 * nanosleep back-off): for ranks sharing one GPU, where a stream blocked in
 * a stream-memory wait can starve the time-sliced context that would raise
 * the flag. */
BP_API int bp_flag_wait_spin(void* stream, const void* addr, uint32_t value);

#ifdef __cplusplus
}
#endif
#endif /* BITPIPE_B200_COMM_H */
