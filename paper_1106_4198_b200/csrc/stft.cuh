// Spectrogram front end (reference audio.hpp:121-187): sine-windowed one-sided
// power spectrum and the silence filter, on the device in fp64.
//   stft_fft_kernel  one CTA per frame, radix-2 decimation-in-time FFT in shared
//                    memory (power-of-two windows up to 4096)
//   stft_dft_kernel  one CTA per frame, direct DFT (any even window)
//   frame_power_kernel / silence_select_kernel  total power per frame (fixed-order
//                    warp sums), the maximum, the -threshold_db floor and the
//                    ascending list of retained frames (deterministic compaction).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace isnmf_dev {

constexpr int kStftThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// tw[m] = exp(-2 pi i m / W), win[i] = sin(pi (i + 0.5) / W) (host fp64 tables)
__global__ void __launch_bounds__(kStftThreads) stft_fft_kernel(const double* samples, int W, int logW, int hop,
                                                                 const double* win, const double2* tw, double* power,
                                                                 int bins) {
  extern __shared__ double2 buf[];  // [W]
  const int n = blockIdx.x, tid = threadIdx.x;
  const double* x = samples + size_t(n) * hop;
  for (int i = tid; i < W; i += kStftThreads) {
    const int r = int(__brev(unsigned(i)) >> (32 - logW));
    buf[r] = make_double2(x[i] * win[i], 0.0);
  }
  __syncthreads();
  for (int s = 1; s <= logW; ++s) {
    const int half = 1 << (s - 1), step = W >> s;
    for (int j = tid; j < W / 2; j += kStftThreads) {
      const int pos = j & (half - 1), i0 = ((j >> (s - 1)) << s) + pos, i1 = i0 + half;
      const double2 t = cmul(tw[pos * step], buf[i1]);
      const double2 u = buf[i0];
      buf[i0] = make_double2(u.x + t.x, u.y + t.y);
      buf[i1] = make_double2(u.x - t.x, u.y - t.y);
    }
    __syncthreads();
  }
  for (int f = tid; f < bins; f += kStftThreads) power[size_t(n) * bins + f] = buf[f].x * buf[f].x + buf[f].y * buf[f].y;
}

__global__ void __launch_bounds__(kStftThreads) stft_dft_kernel(const double* samples, int W, int hop,
                                                                 const double* win, const double2* tw, double* power,
                                                                 int bins) {
  extern __shared__ double xs[];  // [W] windowed frame
  const int n = blockIdx.x, tid = threadIdx.x;
  const double* x = samples + size_t(n) * hop;
  for (int i = tid; i < W; i += kStftThreads) xs[i] = x[i] * win[i];
  __syncthreads();
  for (int f = tid; f < bins; f += kStftThreads) {
    double re = 0.0, im = 0.0;
    int m = 0;  // (f * i) mod W, stepped
    for (int i = 0; i < W; ++i) {
      const double2 w = tw[m];
      re = fma(xs[i], w.x, re);
      im = fma(xs[i], w.y, im);
      m += f;
      if (m >= W) m -= W;
    }
    power[size_t(n) * bins + f] = re * re + im * im;
  }
}

// total power of every frame (one warp per frame, lane-strided then the fixed shuffle tree)
__global__ void frame_power_kernel(const double* spec, int64_t bins, int64_t frames, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t n = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5); n < frames; n += warps) {
    double s = 0.0;
    for (int64_t f = lane; f < bins; f += 32) s += spec[n * bins + f];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[n] = s;
  }
}

constexpr int kSelThreads = 1024;

// one block: max power, the floor, and the ascending indices of the frames at or above it
__global__ void __launch_bounds__(kSelThreads) silence_select_kernel(const double* power, int64_t frames,
                                                                      double threshold_db, int64_t* keep,
                                                                      int64_t* n_keep, int* all_silent) {
  __shared__ double smax[kSelThreads / 32];
  __shared__ int64_t counts[kSelThreads];
  __shared__ double s_floor;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double m = 0.0;
  for (int64_t i = tid; i < frames; i += kSelThreads) m = fmax(m, power[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) smax[warp] = m;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int w = 0; w < kSelThreads / 32; ++w) mx = fmax(mx, smax[w]);
    *all_silent = !(mx > 0.0);
    s_floor = mx * pow(10.0, threshold_db / 10.0);
  }
  __syncthreads();
  const double floor = s_floor;
  const int64_t seg = (frames + kSelThreads - 1) / kSelThreads, b = tid * seg, e = min(frames, b + seg);
  int64_t c = 0;
  for (int64_t i = b; i < e; ++i) c += power[i] >= floor;
  counts[tid] = c;
  __syncthreads();
  if (tid == 0) {  // exclusive scan in thread order
    int64_t run = 0;
    for (int i = 0; i < kSelThreads; ++i) {
      const int64_t v = counts[i];
      counts[i] = run;
      run += v;
    }
    *n_keep = run;
  }
  __syncthreads();
  int64_t o = counts[tid];
  for (int64_t i = b; i < e; ++i)
    if (power[i] >= floor) keep[o++] = i;
}

}  // namespace isnmf_dev
