// detect.cu — F3: the `traffic` application's second stage on
// the device.  SSD-MobileNet-V1 head outputs -> box decode -> per-class greedy
// NMS -> per-image merge -> crops resized for the recognisers.  The
// paper is silent on all of it; the textbook readings are DESIGN.md R27 and
// include/gpulet.h gl_ssd_detect / gl_crop_resize.
//
// Kernels (CUDA cores; the work is a few thousand boxes per image, latency-bound):
//   ssd_nms_kernel    one CTA per (class, image): threshold scan of the class's
//                     3000 scores (strided 84 B, warp-aggregated append), radix
//                     select of the top_k smallest 64-bit (score desc, prior
//                     asc) keys when more pass, bitonic sort of those in smem,
//                     decode of the first top_k, IoU bit-mask rows (one thread
//                     per (i, 32-column word)), then one warp walks the rows
//                     greedily, 32 candidates per block (the mask is the
//                     pairwise suppression relation, the walk is exactly the
//                     sequential greedy NMS).
//   ssd_merge_kernel  8 CTAs per image: the classes' kept lists (each already
//                     sorted) merged on (score desc, class asc, prior asc) by
//                     rank (binary search per class), the first max_det
//                     decoded into [x1, y1, x2, y2, score, class, prior].
//   crop_kernel       one thread per 4 output pixels of one crop: 4 taps of 8
//                     bf16 channels each (16-B loads, all 16 issued before the
//                     arithmetic), bilinear in fp32, bf16 out.
// Arithmetic that decides integers (the score threshold, IoU > thr) or is
// compared bit for bit is written with explicit _rn intrinsics (no FMA
// contraction) in the order R27 states.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gpulet.h"

namespace gl {
gl_status set_error(gl_status s, const char* m);   // runtime.cpp: gl_last_error() text
}

namespace {

constexpr int kPriors = 3000, kClasses = 21, kMaxTopK = 400, kSortCap = 4096;
constexpr int kNmsThreads = 512, kMergeThreads = 256, kMergeSlices = 8;
constexpr int kMaskWords = (kMaxTopK + 31) / 32;
constexpr int kSelCap = 512;   // >= kMaxTopK, power of two: the selected keys
constexpr size_t kNmsSmem = kSortCap * 8 + kSelCap * 8 + kMaxTopK * 16 + (size_t)kMaxTopK * kMaskWords * 4;

// prior p (head order: map, h, w, prior) -> (cx, cy, w, h), fp64 then fp32 (R27)
__device__ void prior_of(int p, float pr[4]) {
  const int maps[6] = {19, 10, 5, 3, 2, 1};
  int k = 0, base = 0;
  while (p >= base + maps[k] * maps[k] * 6) base += maps[k] * maps[k] * 6, ++k;
  const int f = maps[k], r = p - base, cell = r / 6, a = r % 6, i = cell / f, j = cell % f;
  const double sk = 0.2 + 0.75 * k / 5.0, sk1 = k + 1 < 6 ? 0.2 + 0.75 * (k + 1) / 5.0 : 1.0;
  const double cx = (j + 0.5) / f, cy = (i + 0.5) / f;
  double w, h;
  if (a == 5) {
    w = h = sqrt(__dmul_rn(sk, sk1));
  } else {
    const double ar = a == 0 ? 1.0 : a == 1 ? 2.0 : a == 2 ? 0.5 : a == 3 ? 3.0 : 1.0 / 3.0;
    const double rt = sqrt(ar);
    w = __dmul_rn(sk, rt);
    h = __ddiv_rn(sk, rt);
  }
  pr[0] = (float)cx, pr[1] = (float)cy, pr[2] = (float)w, pr[3] = (float)h;
}

__device__ float clip01(float v) { return fminf(fmaxf(v, 0.f), 1.f); }

// decode with variances (0.1, 0.2) in fp64, each operation rounded (R27)
__device__ float4 decode_box(const float* loc4, int p) {
  float pr[4];
  prior_of(p, pr);
  const double pcx = pr[0], pcy = pr[1], pw = pr[2], ph = pr[3];
  const double cx = __dadd_rn(pcx, __dmul_rn(__dmul_rn((double)loc4[0], 0.1), pw));
  const double cy = __dadd_rn(pcy, __dmul_rn(__dmul_rn((double)loc4[1], 0.1), ph));
  const double w = __dmul_rn(pw, exp(__dmul_rn((double)loc4[2], 0.2)));
  const double h = __dmul_rn(ph, exp(__dmul_rn((double)loc4[3], 0.2)));
  const double hw = __dmul_rn(w, 0.5), hh = __dmul_rn(h, 0.5);
  return make_float4(clip01((float)__dsub_rn(cx, hw)), clip01((float)__dsub_rn(cy, hh)),
                     clip01((float)__dadd_rn(cx, hw)), clip01((float)__dadd_rn(cy, hh)));
}

__device__ bool suppresses(float4 a, float4 b, float thr) {
  const float iw = fmaxf(0.f, __fsub_rn(fminf(a.z, b.z), fmaxf(a.x, b.x)));
  const float ih = fmaxf(0.f, __fsub_rn(fminf(a.w, b.w), fmaxf(a.y, b.y)));
  const float inter = __fmul_rn(iw, ih);
  const float area_a = __fmul_rn(__fsub_rn(a.z, a.x), __fsub_rn(a.w, a.y));
  const float area_b = __fmul_rn(__fsub_rn(b.z, b.x), __fsub_rn(b.w, b.y));
  const float uni = __fsub_rn(__fadd_rn(area_a, area_b), inter);
  return __fdiv_rn(inter, uni) > thr;   // NaN (0/0) never suppresses
}

// ascending bitonic sort of n (power of two) 64-bit keys in shared memory
__device__ void bitonic(unsigned long long* key, int n) {
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = key[i], b = key[l];
          const bool up = (i & k) == 0;
          if ((a > b) == up) key[i] = b, key[l] = a;
        }
      }
      __syncthreads();
    }
}

__device__ int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// score > 0 (it passed a threshold >= 0): its bits order like the value
__device__ unsigned long long score_key(float s) { return (unsigned long long)(0xFFFFFFFFu - __float_as_uint(s)) << 32; }

struct Kept {
  float score;
  int prior;
};

__global__ void __launch_bounds__(kNmsThreads) ssd_nms_kernel(const float* __restrict__ loc, const float* __restrict__ conf,
                                                              float score_thr, float iou_thr, int top_k,
                                                              Kept* __restrict__ kept, int* __restrict__ n_kept) {
  extern __shared__ __align__(16) unsigned char nms_smem[];
  unsigned long long* key = (unsigned long long*)nms_smem;     // [kSortCap]
  unsigned long long* sel = key + kSortCap;                  // [kSelCap]
  float4* box = (float4*)(sel + kSelCap);                     // [kMaxTopK]
  uint32_t(*mask)[kMaskWords] = (uint32_t(*)[kMaskWords])(box + kMaxTopK);   // [kMaxTopK][kMaskWords]
  __shared__ int n_cand;
  const int c = blockIdx.x + 1, n = blockIdx.y;
  if (threadIdx.x == 0) n_cand = 0;
  __syncthreads();
  const float* cf = conf + (int64_t)n * kPriors * kClasses + c;
  const int lane = threadIdx.x & 31;
  for (int p0 = threadIdx.x - lane; p0 < kPriors; p0 += blockDim.x) {   // warp-aggregated append
    const int p = p0 + lane;
    const float s = p < kPriors ? __ldg(cf + (int64_t)p * kClasses) : 0.f;
    const bool take = p < kPriors && s > score_thr;
    const uint32_t bal = __ballot_sync(0xffffffffu, take);
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(&n_cand, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (take) key[base + __popc(bal & ((1u << lane) - 1))] = score_key(s) | (unsigned)p;
  }
  __syncthreads();
  const int nc = n_cand, m = min(nc, top_k), words = (m + 31) / 32;
  if (nc > m) {
    // Only the m smallest keys matter: radix-select the m-th smallest key
    // (distinct keys; bits 31..16 are zero) and keep the keys <= it, so the
    // sort below runs on <= 512 keys instead of up to 4096.
    __shared__ uint32_t hist[256];
    __shared__ unsigned long long sel_prefix, sel_mask;
    __shared__ int sel_need, n_sel;
    if (threadIdx.x == 0) sel_prefix = 0, sel_mask = 0, sel_need = m, n_sel = 0;
    const int shifts[6] = {56, 48, 40, 32, 8, 0};
    for (int ps = 0; ps < 6; ++ps) {
      const int sh = shifts[ps];
      for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
      __syncthreads();
      const unsigned long long pre = sel_prefix, msk = sel_mask;
      for (int i = threadIdx.x; i < nc; i += blockDim.x)
        if ((key[i] & msk) == pre) atomicAdd(&hist[(key[i] >> sh) & 255], 1u);
      __syncthreads();
      if (threadIdx.x < 32) {   // warp scan: the digit where the running count reaches sel_need
        uint32_t loc8[8], part = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) loc8[q] = hist[lane * 8 + q], part += loc8[q];
        uint32_t incl = part;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const uint32_t need = (uint32_t)sel_need, excl = incl - part;
        __syncwarp();   // every lane has read sel_need before one lane rewrites it
        if (excl < need && incl >= need) {
          uint32_t run = excl;
          int d = 0;
          while (run + loc8[d] < need) run += loc8[d++];
          sel_prefix = pre | (unsigned long long)(lane * 8 + d) << sh;
          sel_mask = msk | 255ull << sh;
          sel_need = (int)(need - run);
        }
      }
      __syncthreads();
    }
    const unsigned long long kth = sel_prefix;
    for (int i0 = threadIdx.x - lane; i0 < nc; i0 += blockDim.x) {
      const int i = i0 + lane;
      const bool take = i < nc && key[i] <= kth;
      const uint32_t bal = __ballot_sync(0xffffffffu, take);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(&n_sel, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (take) sel[base + __popc(bal & ((1u << lane) - 1))] = key[i];
    }
    __syncthreads();
    key = sel;   // exactly m keys
  }
  const int np2 = pow2_at_least(m);
  for (int i = m + threadIdx.x; i < np2; i += blockDim.x) key[i] = ~0ull;
  __syncthreads();
  bitonic(key, np2);
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    box[i] = decode_box(loc + ((int64_t)n * kPriors + (int)(key[i] & 0xFFFFFFFFu)) * 4, (int)(key[i] & 0xFFFFFFFFu));
  __syncthreads();
  // mask[i] bit j (j > i): candidate j overlaps candidate i above the threshold
  for (int t = threadIdx.x; t < m * words; t += blockDim.x) {
    const int i = t / words, w = t % words;
    if (w < (i >> 5)) continue;   // words left of row i's block are never read by the walk
    uint32_t bits = 0;
    const float4 bi = box[i];
    for (int b = 0; b < 32; ++b) {
      const int j = w * 32 + b;
      if (j > i && j < m && suppresses(bi, box[j], iou_thr)) bits |= 1u << b;
    }
    mask[i][w] = bits;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    // Greedy walk in blocks of 32 candidates: lane w holds word w of the
    // removed set; inside block bk the keep decisions depend only on word bk,
    // resolved with the block's own mask words (shuffled from lane t = row
    // 32 bk + t, independent of the decisions, so the shuffles pipeline);
    // then each lane ORs the kept rows into its later word.
    uint32_t removed = 0;
    int cnt = 0;
    Kept* out = kept + ((int64_t)n * (kClasses - 1) + (c - 1)) * top_k;
    for (int bk = 0; bk < words; ++bk) {
      const int lim = min(32, m - 32 * bk);
      uint32_t rem = __shfl_sync(0xffffffffu, removed, bk), keepbits = 0;
      const uint32_t my = lane < lim ? mask[32 * bk + lane][bk] : 0u;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const uint32_t row = __shfl_sync(0xffffffffu, my, t);
        if (t < lim && !(rem >> t & 1u)) keepbits |= 1u << t, rem |= row;
      }
      for (uint32_t kb = keepbits; kb; kb &= kb - 1)
        if (lane > bk && lane < words) removed |= mask[32 * bk + __ffs(kb) - 1][lane];
      if (keepbits >> lane & 1u) {
        const unsigned long long q = key[32 * bk + lane];
        out[cnt + __popc(keepbits & ((1u << lane) - 1))] =
            Kept{__uint_as_float(0xFFFFFFFFu - (uint32_t)(q >> 32)), (int)(q & 0xFFFFFFFFu)};
      }
      cnt += __popc(keepbits);
    }
    if (lane == 0) n_kept[n * (kClasses - 1) + (c - 1)] = cnt;
  }
}

// merged key of class list entry t of class c: (score desc, class asc, prior asc)
__device__ __forceinline__ unsigned long long merge_key(const Kept& k, int c) {
  return score_key(k.score) | (unsigned long long)(c + 1) << 16 | (unsigned)k.prior;
}

__global__ void __launch_bounds__(kMergeThreads) ssd_merge_kernel(const float* __restrict__ loc, const Kept* __restrict__ kept,
                                                                  const int* __restrict__ n_kept, int top_k, int max_det,
                                                                  float* __restrict__ det, int* __restrict__ count) {
  // Each class list is already in (score desc, prior asc) order, so the merged
  // order needs no sort: an entry's output position is the number of entries
  // of all classes whose merged key is smaller (binary search per class, keys
  // are distinct).  Only each class's first max_det entries can place.
  extern __shared__ unsigned long long mkey[];   // [20][min(top_k, max_det)]
  __shared__ int len[kClasses - 1];
  const int n = blockIdx.x, cap = min(top_k, max_det), S = gridDim.y;
  if (threadIdx.x < kClasses - 1) len[threadIdx.x] = min(n_kept[n * (kClasses - 1) + threadIdx.x], cap);
  __syncthreads();
  for (int t = threadIdx.x; t < (kClasses - 1) * cap; t += blockDim.x) {
    const int c = t / cap, i = t % cap;
    if (i < len[c]) mkey[c * cap + i] = merge_key(kept[((int64_t)n * (kClasses - 1) + c) * top_k + i], c);
  }
  __syncthreads();
  int total = 0;
  for (int c = 0; c < kClasses - 1; ++c) total += len[c];
  for (int t = blockIdx.y * blockDim.x + threadIdx.x; t < (kClasses - 1) * cap; t += S * blockDim.x) {
    const int c = t / cap, i = t % cap;
    if (i >= len[c]) continue;
    const unsigned long long q = mkey[c * cap + i];
    int rank = i;
    for (int c2 = 0; c2 < kClasses - 1 && rank < max_det; ++c2) {
      if (c2 == c) continue;
      int lo = 0, hi = len[c2];   // first entry of class c2 with key > q
      const unsigned long long* L = mkey + c2 * cap;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (L[mid] < q) lo = mid + 1;
        else hi = mid;
      }
      rank += lo;
    }
    if (rank >= max_det) continue;
    const int p = (int)(q & 0xFFFF);
    const float4 b = decode_box(loc + ((int64_t)n * kPriors + p) * 4, p);
    float* o = det + ((int64_t)n * max_det + rank) * 7;
    o[0] = b.x, o[1] = b.y, o[2] = b.z, o[3] = b.w;
    o[4] = __uint_as_float(0xFFFFFFFFu - (uint32_t)(q >> 32));
    o[5] = (float)(c + 1), o[6] = (float)p;
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) count[n] = min(total, max_det);
}

__device__ __forceinline__ float lerp_rn(float a, float b, float w) { return __fadd_rn(a, __fmul_rn(__fsub_rn(b, a), w)); }

constexpr int kCropPix = 4;   // output pixels per thread: the box set-up and 16 tap loads amortised / in flight

__global__ void __launch_bounds__(128) crop_kernel(const __nv_bfloat16* __restrict__ img, int H, int W,
                                                   const float* __restrict__ det, const int* __restrict__ count,
                                                   int max_det, int per_img, int OH, int OW,
                                                   __nv_bfloat16* __restrict__ out) {
  const int crop = blockIdx.y, n = crop / per_img, k = crop % per_img;
  // pixel q of this thread: blockIdx.x * 4 * blockDim + q * blockDim + tid, so
  // one warp store covers 32 consecutive pixels (512 contiguous bytes)
  const int pix0 = blockIdx.x * blockDim.x * kCropPix + threadIdx.x, step = blockDim.x;
  if (pix0 >= OH * OW) return;
  uint4* dst = (uint4*)(out + ((int64_t)crop * OH * OW) * 8);
  if (k >= __ldg(count + n)) {
    for (int q = 0; q < kCropPix && pix0 + q * step < OH * OW; ++q) dst[pix0 + q * step] = make_uint4(0, 0, 0, 0);
    return;
  }
  const float* d = det + ((int64_t)n * max_det + k) * 7;
  const float x1 = __ldg(d), y1 = __ldg(d + 1), x2 = __ldg(d + 2), y2 = __ldg(d + 3);
  const float fW = (float)W, fH = (float)H;
  const float sw = __fdiv_rn(__fmul_rn(__fsub_rn(x2, x1), fW), (float)OW);
  const float sh = __fdiv_rn(__fmul_rn(__fsub_rn(y2, y1), fH), (float)OH);
  const uint4* base = (const uint4*)(img + (int64_t)n * H * W * 8);
  uint4 q4[kCropPix][4];
  float wxs[kCropPix], wys[kCropPix];
#pragma unroll
  for (int q = 0; q < kCropPix; ++q) {   // issue all tap loads first
    const int pix = min(pix0 + q * step, OH * OW - 1), oy = pix / OW, ox = pix % OW;
    float sy = __fsub_rn(__fadd_rn(__fmul_rn(y1, fH), __fmul_rn(__fadd_rn((float)oy, 0.5f), sh)), 0.5f);
    float sx = __fsub_rn(__fadd_rn(__fmul_rn(x1, fW), __fmul_rn(__fadd_rn((float)ox, 0.5f), sw)), 0.5f);
    sy = fminf(fmaxf(sy, 0.f), (float)(H - 1));
    sx = fminf(fmaxf(sx, 0.f), (float)(W - 1));
    const int y0 = (int)floorf(sy), x0 = (int)floorf(sx), y1i = min(y0 + 1, H - 1), x1i = min(x0 + 1, W - 1);
    wys[q] = __fsub_rn(sy, (float)y0), wxs[q] = __fsub_rn(sx, (float)x0);
    q4[q][0] = __ldg(base + y0 * W + x0), q4[q][1] = __ldg(base + y0 * W + x1i);
    q4[q][2] = __ldg(base + y1i * W + x0), q4[q][3] = __ldg(base + y1i * W + x1i);
  }
#pragma unroll
  for (int q = 0; q < kCropPix; ++q) {
    if (pix0 + q * step >= OH * OW) break;
    const __nv_bfloat16 *v0 = (const __nv_bfloat16*)&q4[q][0], *v1 = (const __nv_bfloat16*)&q4[q][1],
                        *v2 = (const __nv_bfloat16*)&q4[q][2], *v3 = (const __nv_bfloat16*)&q4[q][3];
    uint4 r;
    __nv_bfloat16* rb = (__nv_bfloat16*)&r;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      const float top = lerp_rn(__bfloat162float(v0[ch]), __bfloat162float(v1[ch]), wxs[q]);
      const float bot = lerp_rn(__bfloat162float(v2[ch]), __bfloat162float(v3[ch]), wxs[q]);
      rb[ch] = __float2bfloat16_rn(lerp_rn(top, bot, wys[q]));
    }
    dst[pix0 + q * step] = r;
  }
}

gl_status cuda_status() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GL_OK : gl::set_error(GL_E_CUDA, cudaGetErrorString(e));
}

gl_status bad(const char* m) { return gl::set_error(GL_E_ARG, m); }

}  // namespace

extern "C" gl_status gl_ssd_detect_workspace(int32_t n_img, int32_t top_k, size_t* bytes) {
  if (!bytes || n_img < 0 || top_k < 1 || top_k > kMaxTopK) return bad("gl_ssd_detect_workspace: n_img >= 0, 1 <= top_k <= 400");
  *bytes = (size_t)n_img * (kClasses - 1) * ((size_t)top_k * sizeof(Kept) + sizeof(int));
  return GL_OK;
}

extern "C" gl_status gl_ssd_detect(const float* loc_dev, const float* conf_dev, int32_t n_img, float score_thr,
                                   float iou_thr, int32_t top_k, int32_t max_det, float* det_dev, int32_t* count_dev,
                                   void* ws_dev, size_t ws_bytes, void* stream) {
  size_t need = 0;
  if (gl_ssd_detect_workspace(n_img, top_k, &need) != GL_OK || max_det < 1 || !(score_thr >= 0.f) ||
      !(iou_thr >= 0.f))
    return bad("gl_ssd_detect: n_img >= 0, 1 <= top_k <= 400, max_det >= 1, thresholds >= 0");
  if (n_img == 0) return GL_OK;
  if (!loc_dev || !conf_dev || !det_dev || !count_dev || !ws_dev) return bad("gl_ssd_detect: null pointer");
  if (ws_bytes < need) return bad("gl_ssd_detect: workspace smaller than gl_ssd_detect_workspace()");
  cudaStream_t s = (cudaStream_t)stream;
  Kept* kept = (Kept*)ws_dev;
  int* n_kept = (int*)(kept + (size_t)n_img * (kClasses - 1) * top_k);
  static const cudaError_t attr_nms =   // once per process (a host call between the two launches would show as a gap)
      cudaFuncSetAttribute(ssd_nms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNmsSmem);
  static const cudaError_t attr_merge = cudaFuncSetAttribute(
      ssd_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (kClasses - 1) * kMaxTopK * 8);
  if (attr_nms != cudaSuccess || attr_merge != cudaSuccess) return gl::set_error(GL_E_CUDA, "gl_ssd_detect: smem attribute");
  ssd_nms_kernel<<<dim3(kClasses - 1, n_img), kNmsThreads, kNmsSmem, s>>>(loc_dev, conf_dev, score_thr, iou_thr, top_k, kept,
                                                                   n_kept);
  const int cap = (kClasses - 1) * (top_k < max_det ? top_k : max_det);   // <= 8000 keys
  ssd_merge_kernel<<<dim3(n_img, kMergeSlices), kMergeThreads, (size_t)cap * 8, s>>>(loc_dev, kept, n_kept, top_k, max_det, det_dev,
                                                                  count_dev);
  return cuda_status();
}

extern "C" gl_status gl_crop_resize(const void* img_dev, int32_t n_img, int32_t H, int32_t W, int32_t C,
                                    const float* det_dev, const int32_t* count_dev, int32_t max_det, int32_t per_img,
                                    int32_t OH, int32_t OW, void* out_dev, void* stream) {
  if (n_img < 0 || H < 1 || W < 1 || C != 8 || per_img < 1 || per_img > max_det || OH < 1 || OW < 1)
    return bad("gl_crop_resize: n_img >= 0, H, W, OH, OW >= 1, C == 8, 1 <= per_img <= max_det");
  if (n_img == 0) return GL_OK;
  if (!img_dev || !det_dev || !count_dev || !out_dev) return bad("gl_crop_resize: null pointer");
  const int threads = 128;
  const int per_block = threads * kCropPix;
  crop_kernel<<<dim3((OH * OW + per_block - 1) / per_block, n_img * per_img), threads, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)img_dev, H, W, det_dev, count_dev, max_det, per_img, OH, OW, (__nv_bfloat16*)out_dev);
  return cuda_status();
}
