// detect.cu — F3: the `traffic` application's second stage on
// the device.  SSD-MobileNet-V1 head outputs -> box decode -> per-class greedy
// NMS -> per-image merge -> crops resized for the recognisers.  The
// paper is silent on all of it; the textbook readings are DESIGN.md R27 and
// include/gpulet.h gl_ssd_detect / gl_crop_resize.
//
// Kernels (CUDA cores; the work is a few thousand boxes per image, latency-bound):
//   ssd_nms_kernel    one CTA per (class, image): threshold scan of the class's
//                     3000 scores (strided 84 B), bitonic sort of the candidates
//                     on a 64-bit (score desc, prior asc) key in shared memory,
//                     decode of the first top_k, IoU bit-mask rows (one thread
//                     per (i, 32-column word)), then one warp walks the rows
//                     greedily (the mask is the pairwise suppression relation,
//                     the walk is exactly the sequential greedy NMS).
//   ssd_merge_kernel  one CTA per image: the classes' kept lists sorted on
//                     (score desc, class asc, prior asc), first max_det decoded
//                     into [x1, y1, x2, y2, score, class, prior].
//   crop_kernel       one thread per output pixel of one crop: 4 taps of 8
//                     bf16 channels (16-B loads), bilinear in fp32, bf16 out.
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

constexpr int kPriors = 3000, kClasses = 21, kMaxTopK = 400, kSortCap = 4096, kMergeCap = 8192;
constexpr int kNmsThreads = 512, kMergeThreads = 1024;
constexpr int kMaskWords = (kMaxTopK + 31) / 32;
constexpr size_t kNmsSmem = kSortCap * 8 + kMaxTopK * 16 + (size_t)kMaxTopK * kMaskWords * 4;

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
  float4* box = (float4*)(key + kSortCap);                    // [kMaxTopK]
  uint32_t(*mask)[kMaskWords] = (uint32_t(*)[kMaskWords])(box + kMaxTopK);   // [kMaxTopK][kMaskWords]
  __shared__ int n_cand;
  const int c = blockIdx.x + 1, n = blockIdx.y;
  if (threadIdx.x == 0) n_cand = 0;
  __syncthreads();
  const float* cf = conf + (int64_t)n * kPriors * kClasses + c;
  for (int p = threadIdx.x; p < kPriors; p += blockDim.x) {
    const float s = __ldg(cf + (int64_t)p * kClasses);
    if (s > score_thr) key[atomicAdd(&n_cand, 1)] = score_key(s) | (unsigned)p;
  }
  __syncthreads();
  const int nc = n_cand, np2 = pow2_at_least(nc);
  for (int i = nc + threadIdx.x; i < np2; i += blockDim.x) key[i] = ~0ull;
  __syncthreads();
  bitonic(key, np2);
  const int m = min(nc, top_k), words = (m + 31) / 32;
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    box[i] = decode_box(loc + ((int64_t)n * kPriors + (int)(key[i] & 0xFFFFFFFFu)) * 4, (int)(key[i] & 0xFFFFFFFFu));
  __syncthreads();
  // mask[i] bit j (j > i): candidate j overlaps candidate i above the threshold
  for (int t = threadIdx.x; t < m * words; t += blockDim.x) {
    const int i = t / words, w = t % words;
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
    const int lane = threadIdx.x;
    uint32_t removed = 0;   // this lane's word of the removed set: words lane (m <= 400 -> 13 words)
    int cnt = 0;
    Kept* out = kept + ((int64_t)n * (kClasses - 1) + (c - 1)) * top_k;
    for (int i = 0; i < m; ++i) {
      const uint32_t word = __shfl_sync(0xffffffffu, removed, i >> 5);
      if (word >> (i & 31) & 1u) continue;
      if (lane == 0) out[cnt] = Kept{__uint_as_float(0xFFFFFFFFu - (uint32_t)(key[i] >> 32)), (int)(key[i] & 0xFFFFFFFFu)};
      ++cnt;
      if (lane < words) removed |= mask[i][lane];
    }
    if (lane == 0) n_kept[n * (kClasses - 1) + (c - 1)] = cnt;
  }
}

__global__ void __launch_bounds__(kMergeThreads) ssd_merge_kernel(const float* __restrict__ loc, const Kept* __restrict__ kept,
                                                                  const int* __restrict__ n_kept, int top_k, int max_det,
                                                                  float* __restrict__ det, int* __restrict__ count) {
  extern __shared__ unsigned long long mkey[];
  __shared__ int off[kClasses];
  const int n = blockIdx.x;
  if (threadIdx.x == 0) {
    int s = 0;
    for (int c = 0; c < kClasses - 1; ++c) off[c] = s, s += n_kept[n * (kClasses - 1) + c];
    off[kClasses - 1] = s;
  }
  __syncthreads();
  const int total = off[kClasses - 1], np2 = pow2_at_least(total);
  for (int c = 0; c < kClasses - 1; ++c) {
    const Kept* src = kept + ((int64_t)n * (kClasses - 1) + c) * top_k;
    for (int t = threadIdx.x; t < off[c + 1] - off[c]; t += blockDim.x)
      mkey[off[c] + t] = score_key(src[t].score) | (unsigned long long)(c + 1) << 16 | (unsigned)src[t].prior;
  }
  for (int i = total + threadIdx.x; i < np2; i += blockDim.x) mkey[i] = ~0ull;
  __syncthreads();
  bitonic(mkey, np2);
  const int nd = min(total, max_det);
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    const unsigned long long q = mkey[k];
    const int p = (int)(q & 0xFFFF), c = (int)(q >> 16 & 0xFFFF);
    const float4 b = decode_box(loc + ((int64_t)n * kPriors + p) * 4, p);
    float* o = det + ((int64_t)n * max_det + k) * 7;
    o[0] = b.x, o[1] = b.y, o[2] = b.z, o[3] = b.w;
    o[4] = __uint_as_float(0xFFFFFFFFu - (uint32_t)(q >> 32));
    o[5] = (float)c, o[6] = (float)p;
  }
  if (threadIdx.x == 0) count[n] = nd;
}

__device__ __forceinline__ float lerp_rn(float a, float b, float w) { return __fadd_rn(a, __fmul_rn(__fsub_rn(b, a), w)); }

__global__ void crop_kernel(const __nv_bfloat16* __restrict__ img, int H, int W, const float* __restrict__ det,
                            const int* __restrict__ count, int max_det, int per_img, int OH, int OW,
                            __nv_bfloat16* __restrict__ out) {
  const int crop = blockIdx.y, n = crop / per_img, k = crop % per_img;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= OH * OW) return;
  const int oy = pix / OW, ox = pix % OW;
  uint4* dst = (uint4*)(out + ((int64_t)crop * OH * OW + pix) * 8);
  if (k >= count[n]) {
    *dst = make_uint4(0, 0, 0, 0);
    return;
  }
  const float* d = det + ((int64_t)n * max_det + k) * 7;
  const float x1 = d[0], y1 = d[1], x2 = d[2], y2 = d[3];
  const float fW = (float)W, fH = (float)H;
  const float sw = __fdiv_rn(__fmul_rn(__fsub_rn(x2, x1), fW), (float)OW);
  const float sh = __fdiv_rn(__fmul_rn(__fsub_rn(y2, y1), fH), (float)OH);
  float sy = __fsub_rn(__fadd_rn(__fmul_rn(y1, fH), __fmul_rn(__fadd_rn((float)oy, 0.5f), sh)), 0.5f);
  float sx = __fsub_rn(__fadd_rn(__fmul_rn(x1, fW), __fmul_rn(__fadd_rn((float)ox, 0.5f), sw)), 0.5f);
  sy = fminf(fmaxf(sy, 0.f), (float)(H - 1));
  sx = fminf(fmaxf(sx, 0.f), (float)(W - 1));
  const int y0 = (int)floorf(sy), x0 = (int)floorf(sx), y1i = min(y0 + 1, H - 1), x1i = min(x0 + 1, W - 1);
  const float wy = __fsub_rn(sy, (float)y0), wx = __fsub_rn(sx, (float)x0);
  const uint4* base = (const uint4*)(img + (int64_t)n * H * W * 8);
  uint4 q[4] = {__ldg(base + y0 * W + x0), __ldg(base + y0 * W + x1i), __ldg(base + y1i * W + x0),
                __ldg(base + y1i * W + x1i)};
  const __nv_bfloat16* v[4] = {(const __nv_bfloat16*)&q[0], (const __nv_bfloat16*)&q[1], (const __nv_bfloat16*)&q[2],
                               (const __nv_bfloat16*)&q[3]};
  uint4 r;
  __nv_bfloat16* rb = (__nv_bfloat16*)&r;
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    const float top = lerp_rn(__bfloat162float(v[0][ch]), __bfloat162float(v[1][ch]), wx);
    const float bot = lerp_rn(__bfloat162float(v[2][ch]), __bfloat162float(v[3][ch]), wx);
    rb[ch] = __float2bfloat16_rn(lerp_rn(top, bot, wy));
  }
  *dst = r;
}

int pow2_host(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
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
  cudaFuncSetAttribute(ssd_nms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNmsSmem);
  cudaFuncSetAttribute(ssd_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMergeCap * 8);
  ssd_nms_kernel<<<dim3(kClasses - 1, n_img), kNmsThreads, kNmsSmem, s>>>(loc_dev, conf_dev, score_thr, iou_thr, top_k, kept,
                                                                   n_kept);
  const int cap = pow2_host((kClasses - 1) * top_k);
  ssd_merge_kernel<<<n_img, kMergeThreads, (size_t)cap * 8, s>>>(loc_dev, kept, n_kept, top_k, max_det, det_dev,
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
  crop_kernel<<<dim3((OH * OW + threads - 1) / threads, n_img * per_img), threads, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)img_dev, H, W, det_dev, count_dev, max_det, per_img, OH, OW, (__nv_bfloat16*)out_dev);
  return cuda_status();
}
