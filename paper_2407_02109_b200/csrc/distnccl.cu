// pscwin_dist_forward: one PSCWin layer on this rank's band of window rows of one
// image, with the three exchanges of the band path done IN the library over NCCL on the caller's stream (NVLink /
// NVSwitch on the box): the conv-history ring (k-1 xin rows), the all-gather of the per-rank scan records
// (SURVEY Appendix A fold), and the QKV halo rows of the shifted windows that straddle a band edge. The phases are
// the pscwin_band_* calls; everything is stream-ordered, so the whole layer (exchanges included) can be captured in
// a CUDA graph. Communicators come from the caller (any ncclComm_t) or from pscwin_nccl_comm_init.
#include <nccl.h>
#include <string.h>

#include <chrono>
#include <thread>

#include "../../include/pscwin.h"
#include "pscwin_internal.h"

namespace {
inline uint8_t* at(void* ws, uint64_t off) { return reinterpret_cast<uint8_t*>(ws) + off; }
inline int nccl_ok(ncclResult_t r) { return r == ncclSuccess ? PSCWIN_OK : PSCWIN_ERR_NCCL; }
}  // namespace

extern "C" {

int pscwin_nccl_get_unique_id(void* id_out) {
  if (!id_out) return PSCWIN_ERR_SHAPE;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PSCWIN_ERR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return PSCWIN_OK;
}

int pscwin_nccl_comm_init(const void* id_in, int32_t world, int32_t rank, void** comm_out) {
  if (!id_in || !comm_out || world < 1 || rank < 0 || rank >= world) return PSCWIN_ERR_SHAPE;
  ncclUniqueId id;
  memcpy(&id, id_in, sizeof(id));
  ncclComm_t c = nullptr;
  if (ncclCommInitRank(&c, world, id, rank) != ncclSuccess) return PSCWIN_ERR_NCCL;
  *comm_out = c;
  return PSCWIN_OK;
}

int pscwin_nccl_comm_destroy(void* comm) {
  if (!comm) return PSCWIN_OK;
  return nccl_ok(ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)));
}

int pscwin_nccl_comm_check(void* comm) {
  if (!comm) return PSCWIN_ERR_SHAPE;
  ncclResult_t async = ncclSuccess;
  if (ncclCommGetAsyncError(reinterpret_cast<ncclComm_t>(comm), &async) != ncclSuccess) return PSCWIN_ERR_NCCL;
  return (async == ncclSuccess || async == ncclInProgress) ? PSCWIN_OK : PSCWIN_ERR_NCCL;
}

int pscwin_nccl_comm_abort(void* comm) {
  if (!comm) return PSCWIN_ERR_SHAPE;
  return nccl_ok(ncclCommAbort(reinterpret_cast<ncclComm_t>(comm)));
}

int pscwin_nccl_wait(void* comm, void* stream, int64_t timeout_ms) {
  if (!comm) return PSCWIN_ERR_SHAPE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return PSCWIN_OK;
    if (q != cudaErrorNotReady) return PSCWIN_ERR_CUDA;
    if (pscwin_nccl_comm_check(comm) != PSCWIN_OK) {
      ncclCommAbort(reinterpret_cast<ncclComm_t>(comm));
      return PSCWIN_ERR_NCCL;
    }
    if (timeout_ms > 0 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) {
      ncclCommAbort(reinterpret_cast<ncclComm_t>(comm));
      return PSCWIN_ERR_TIMEOUT;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
}

size_t pscwin_dist_workspace_bytes(const pscwin_layer_desc* d, int32_t row_begin, int32_t row_end, int32_t rank,
                                   int32_t world) {
  pscwin_band b;
  b.row_begin = row_begin;
  b.row_end = row_end;
  b.rank = rank;
  b.world = world;
  return pscwin_band_workspace_bytes(d, &b);
}

static int dist_forward_on(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x_band,
                           void* x_band_out, int32_t row_begin, int32_t row_end, void* nccl_comm, void* ws,
                           size_t ws_bytes, void* stream, void* comm_stream);

int pscwin_dist_forward(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x_band,
                        void* x_band_out, int32_t row_begin, int32_t row_end, void* nccl_comm, void* ws,
                        size_t ws_bytes, void* stream, void* comm_stream) {
  if (stream)
    return dist_forward_on(d, wt, x_band, x_band_out, row_begin, row_end, nccl_comm, ws, ws_bytes, stream,
                           comm_stream);
  // the legacy default stream: NCCL's send / recv to self have been seen to stall there, so the layer runs on a
  // library-owned non-blocking stream (per thread and device, aux_stream slot 1) joined to it by events
  pscwin::AuxStream* own = pscwin::aux_stream(1);
  if (!own) return PSCWIN_ERR_CUDA;
  if (cudaEventRecord(own->fork, 0) != cudaSuccess || cudaStreamWaitEvent(own->s, own->fork, 0) != cudaSuccess)
    return PSCWIN_ERR_CUDA;
  const int rc = dist_forward_on(d, wt, x_band, x_band_out, row_begin, row_end, nccl_comm, ws, ws_bytes, own->s,
                                 comm_stream);
  if (cudaEventRecord(own->join, own->s) != cudaSuccess || cudaStreamWaitEvent(0, own->join, 0) != cudaSuccess)
    return PSCWIN_ERR_CUDA;
  return rc;
}

static int dist_forward_on(const pscwin_layer_desc* d, const pscwin_layer_weights* wt, const void* x_band,
                           void* x_band_out, int32_t row_begin, int32_t row_end, void* nccl_comm, void* ws,
                           size_t ws_bytes, void* stream, void* comm_stream) {
  if (!nccl_comm) return PSCWIN_ERR_SHAPE;
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  // a communicator that already carries an asynchronous error (a peer failed, or it was aborted) would hang or fail
  // inside the enqueued operations: refuse up front
  if (pscwin_nccl_comm_check(nccl_comm) != PSCWIN_OK) return PSCWIN_ERR_NCCL;
  int rank = 0, world = 1;
  if (ncclCommUserRank(comm, &rank) != ncclSuccess || ncclCommCount(comm, &world) != ncclSuccess)
    return PSCWIN_ERR_NCCL;
  pscwin_band b;
  b.row_begin = row_begin;
  b.row_end = row_end;
  b.rank = rank;
  b.world = world;
  pscwin_band_io io;
  int rc = pscwin_band_io_offsets(d, &b, &io);
  if (rc) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int prev = (rank - 1 + world) % world, next = (rank + 1) % world;
  if (d->cycle_scan) {
    // The two scan exchanges are latency-sized (k - 1 xin rows; one record of D (N + 2) floats per rank) and the
    // work after each depends on them (the band's first conv rows; every chunk's entry state), so they stay on the
    // compute stream.
    rc = pscwin_band_scan_begin(d, &b, wt, x_band, ws, ws_bytes, stream);
    if (rc) return rc;
    // conv history ring: rank g -> g+1 (rank 0 receives the global sequence tail from the last rank)
    if (ncclGroupStart() != ncclSuccess) return PSCWIN_ERR_NCCL;
    ncclSend(at(ws, io.hist_send), io.hist_bytes, ncclUint8, next, comm, s);
    ncclRecv(at(ws, io.hist_recv), io.hist_bytes, ncclUint8, prev, comm, s);
    if (ncclGroupEnd() != ncclSuccess) return PSCWIN_ERR_NCCL;
    rc = pscwin_band_scan_mid(d, &b, wt, ws, ws_bytes, stream);
    if (rc) return rc;
    // scan records: all-gather in rank order, then every rank folds them locally (band_scan_end)
    rc = nccl_ok(ncclAllGather(at(ws, io.rec_send), at(ws, io.rec_recv), io.rec_bytes, ncclUint8, comm, s));
    if (rc) return rc;
    rc = pscwin_band_scan_end(d, &b, wt, x_band, ws, ws_bytes, stream);
    if (rc) return rc;
  }
  rc = pscwin_band_attn_begin(d, &b, wt, x_band, ws, ws_bytes, stream);
  if (rc) return rc;
  // QKV halo rows of the shifted windows straddling the band edges (sizes are 0 for plain layers / image edges)
  const bool halo = io.send_prev_bytes || io.send_next_bytes || io.recv_prev_bytes || io.recv_next_bytes;
  cudaStream_t c = reinterpret_cast<cudaStream_t>(comm_stream);
  pscwin::AuxStream* ev = (halo && c && c != s) ? pscwin::aux_stream(2) : nullptr;
  cudaStream_t hs = ev ? c : s;  // the stream the halo exchange runs on
  if (ev) {  // the exchange waits for this band's QKV rows; interior windows run meanwhile on the compute stream
    if (cudaEventRecord(ev->fork, s) != cudaSuccess || cudaStreamWaitEvent(c, ev->fork, 0) != cudaSuccess)
      return PSCWIN_ERR_CUDA;
  }
  if (halo) {
    if (ncclGroupStart() != ncclSuccess) return PSCWIN_ERR_NCCL;
    if (io.send_prev_bytes) ncclSend(at(ws, io.send_prev), io.send_prev_bytes, ncclUint8, rank - 1, comm, hs);
    if (io.send_next_bytes) ncclSend(at(ws, io.send_next), io.send_next_bytes, ncclUint8, rank + 1, comm, hs);
    if (io.recv_prev_bytes) ncclRecv(at(ws, io.recv_prev), io.recv_prev_bytes, ncclUint8, rank - 1, comm, hs);
    if (io.recv_next_bytes) ncclRecv(at(ws, io.recv_next), io.recv_next_bytes, ncclUint8, rank + 1, comm, hs);
    if (ncclGroupEnd() != ncclSuccess) return PSCWIN_ERR_NCCL;
  }
  if (ev) {
    if (cudaEventRecord(ev->join, c) != cudaSuccess) return PSCWIN_ERR_CUDA;
    int top = 0, bot = 0, nwy = 0;
    pscwin::band_window_rows(d, &b, &top, &bot, &nwy);
    if (bot > top) {  // interior window rows: no halo row inside
      rc = pscwin::band_attention(d, &b, wt, ws, ws_bytes, top, bot, 0, stream);
      if (rc) return rc;
    }
    if (cudaStreamWaitEvent(s, ev->join, 0) != cudaSuccess) return PSCWIN_ERR_CUDA;
    // the window rows that read halo rows (the pad tables, if any, were written by the interior launch)
    const int tab = bot > top ? 1 : 0;
    if (top > 0 && (rc = pscwin::band_attention(d, &b, wt, ws, ws_bytes, 0, top, tab, stream))) return rc;
    if (bot < nwy && bot >= top &&
        (rc = pscwin::band_attention(d, &b, wt, ws, ws_bytes, bot, nwy, tab || top > 0, stream)))
      return rc;
    return pscwin::band_out_proj(d, &b, wt, x_band, x_band_out, ws, ws_bytes, stream);
  }
  return pscwin_band_attn_end(d, &b, wt, x_band, x_band_out, ws, ws_bytes, stream);
}

}  // extern "C"
