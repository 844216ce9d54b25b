// Window partition / padded-shift partition / merge (§3.2 P:L110, L116-119;
// App. C). Pure data movement: bit-exact by construction.
//
// Layouts (row-major, contiguous): grid x [B,H,W,Cx]; windows [B*nW, w*w, Cx] with windows row-major over
// (wy,wx) and slots row-major over (iy,ix) (reading Q4). Slot (iy,ix) of window (wy,wx) holds grid
// token (wy*w+iy-pt, wx*w+ix-pl) or, outside the grid, the pad row (pt,pl = (w - s) mod w, reading Q7).
//
// One warp moves one Cx-row with 16-byte vectors (coalesced; 3 iterations for Cx=768 bf16). The merge is
// written as a gather over OUTPUT rows so every output element is written exactly once (no atomics).
#include "common.cuh"
#include "pscwin_internal.h"

namespace pscwin {

struct Geometry {
  int B, H, W, w, pt, pl, nwx, nw;  // nw = windows per image
};

template <typename VecT>
__global__ void partition_kernel(const VecT* __restrict__ x, const VecT* __restrict__ pad_row, VecT* __restrict__ out,
                                 Geometry g, int vecs_per_row, long long n_rows) {
  pdl_trigger();
  pdl_wait();
  long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_rows) return;
  int lane = threadIdx.x & 31;
  int ww = g.w * g.w;
  long long per_img = (long long)g.nw * ww;
  int b = (int)(row / per_img);
  int r = (int)(row - (long long)b * per_img);
  int win = r / ww, slot = r - win * ww;
  int wy = win / g.nwx, wx = win - wy * g.nwx;
  int iy = slot / g.w, ix = slot - iy * g.w;
  int y = wy * g.w + iy - g.pt, xx = wx * g.w + ix - g.pl;
  const VecT* src = (y >= 0 && y < g.H && xx >= 0 && xx < g.W)
                        ? x + (((long long)b * g.H + y) * g.W + xx) * vecs_per_row
                        : pad_row;
  VecT* dst = out + row * vecs_per_row;
  for (int i = lane; i < vecs_per_row; i += 32) dst[i] = src[i];
}

// out[b,y,x,:] = win[b, window(y,x), slot(y,x), :] (+ residual[b,y,x,:]); T = storage element type.
template <typename T>
__global__ void merge_kernel(const T* __restrict__ win, const T* __restrict__ residual, T* __restrict__ out, Geometry g,
                             int Cx, long long n_rows) {
  pdl_trigger();
  pdl_wait();
  long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_rows) return;
  int lane = threadIdx.x & 31;
  long long hw = (long long)g.H * g.W;
  int b = (int)(row / hw);
  int t = (int)(row - b * hw);
  int y = t / g.W, xx = t - y * g.W;
  int Y = y + g.pt, X = xx + g.pl;
  int wy = Y / g.w, wx = X / g.w;
  int slot = (Y - wy * g.w) * g.w + (X - wx * g.w);
  long long src_row = ((long long)b * g.nw + wy * g.nwx + wx) * g.w * g.w + slot;
  const T* src = win + src_row * Cx;
  T* dst = out + row * Cx;
  if (Cx % 8 == 0 && sizeof(T) == 2) {
    // bf16: 8 elements per 16-byte vector
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const uint4* r4 = residual ? reinterpret_cast<const uint4*>(residual + row * Cx) : nullptr;
    for (int i = lane; i < Cx / 8; i += 32) {
      uint4 v = s4[i];
      if (r4) {
        uint4 r = r4[i];
        uint32_t* pv = reinterpret_cast<uint32_t*>(&v);
        const uint32_t* pr = reinterpret_cast<const uint32_t*>(&r);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          pv[j] = pack_bf16(bf16_lo(pv[j]) + bf16_lo(pr[j]), bf16_hi(pv[j]) + bf16_hi(pr[j]));
      }
      d4[i] = v;
    }
  } else {
    for (int i = lane; i < Cx; i += 32) {
      T v = src[i];
      if (residual) {
        if constexpr (sizeof(T) == 4) {
          v = v + residual[row * Cx + i];
        } else {
          v = __float2bfloat16_rn(__bfloat162float(v) + __bfloat162float(residual[row * Cx + i]));
        }
      }
      dst[i] = v;
    }
  }
}

static Geometry make_geometry(int B, int H, int W, int w, int sx, int sy) {
  Geometry g;
  g.B = B;
  g.H = H;
  g.W = W;
  g.w = w;
  g.pl = (w - sx) % w;
  g.pt = (w - sy) % w;
  int pr = ((-(g.pl + W)) % w + w) % w;
  int pb = ((-(g.pt + H)) % w + w) % w;
  g.nwx = (g.pl + W + pr) / w;
  g.nw = ((g.pt + H + pb) / w) * g.nwx;
  return g;
}

int launch_partition(const void* x, const void* pad_row, int B, int H, int W, int Cx, int w, int sx, int sy,
                     int esize, void* out, cudaStream_t stream) {
  Geometry g = make_geometry(B, H, W, w, sx, sy);
  long long n_rows = (long long)B * g.nw * w * w;
  if (n_rows == 0) return 0;
  int rows_per_block = 8;
  unsigned grid = (unsigned)((n_rows + rows_per_block - 1) / rows_per_block);
  size_t row_bytes = (size_t)Cx * esize;
  bool vec16 = row_bytes % 16 == 0 && ((uintptr_t)x % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
               (pad_row == nullptr || (uintptr_t)pad_row % 16 == 0);
  PSCWIN_PROF("partition", stream);
  if (vec16) {
    launch_k(partition_kernel<uint4>, dim3(grid), dim3(256), 0, stream, (const uint4*)x, (const uint4*)pad_row, (uint4*)out, g,
                                                      (int)(row_bytes / 16), n_rows);
  } else if (row_bytes % 4 == 0) {
    launch_k(partition_kernel<uint32_t>, dim3(grid), dim3(256), 0, stream, (const uint32_t*)x, (const uint32_t*)pad_row,
                                                         (uint32_t*)out, g, (int)(row_bytes / 4), n_rows);
  } else {
    launch_k(partition_kernel<uint16_t>, dim3(grid), dim3(256), 0, stream, (const uint16_t*)x, (const uint16_t*)pad_row,
                                                         (uint16_t*)out, g, (int)(row_bytes / 2), n_rows);
  }
  return (int)cudaGetLastError();
}

int launch_merge(const void* win, int B, int H, int W, int Cx, int w, int sx, int sy, const void* residual,
                 int is_f32, void* out, cudaStream_t stream) {
  Geometry g = make_geometry(B, H, W, w, sx, sy);
  long long n_rows = (long long)B * H * W;
  if (n_rows == 0) return 0;
  unsigned grid = (unsigned)((n_rows + 7) / 8);
  PSCWIN_PROF("merge", stream);
  if (is_f32) {
    launch_k(merge_kernel<float>, dim3(grid), dim3(256), 0, stream, (const float*)win, (const float*)residual, (float*)out, g, Cx,
                                                  n_rows);
  } else {
    launch_k(merge_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, stream, (const __nv_bfloat16*)win,
                                                          (const __nv_bfloat16*)residual, (__nv_bfloat16*)out, g,
                                                          Cx, n_rows);
  }
  return (int)cudaGetLastError();
}

}  // namespace pscwin
