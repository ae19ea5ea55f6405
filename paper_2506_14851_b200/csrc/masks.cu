// Correlation masks for sm_100a.
#include "common.cuh"

// ---------------------------------------------------------------------------
// Correlation masks: estimator.pearson (62-81) over
// the (unit, mask) pairs of build_masks (108-142).  One thread per pair runs
// the reference's operation sequence: CPython sum() (Neumaier-compensated,
// in record order) for the means and the centred sums, then
// sxy / sqrt(sxx * syy) clamped to [-1, 1].  The squares are d * d where the
// reference evaluates d ** 2 through libm pow(), which can differ by one ulp,
// so rho agrees to ~1e-15 and the flags agree away from the threshold.
// ---------------------------------------------------------------------------
namespace pdg {
struct Neumaier {
  double f = 0.0, c = 0.0;
  bool first = true;
  __device__ __forceinline__ void add(double x) {
    if (first) { f = dadd(0.0, x); first = false; return; }   // sum() starts at 0 + x0
    const double t = dadd(f, x);
    c = fabs(f) >= fabs(x) ? dadd(c, dadd(dsub(f, t), x)) : dadd(c, dadd(dsub(x, t), f));
    f = t;
  }
  __device__ __forceinline__ double value() const {
    return (c != 0.0 && isfinite(c)) ? dadd(f, c) : f;
  }
};

__global__ void pearson_kernel(const double* __restrict__ x, const double* __restrict__ y,
                               const int32_t* __restrict__ off, const int32_t* __restrict__ len,
                               int64_t n_jobs, double threshold, double* __restrict__ rho,
                               uint8_t* __restrict__ flag) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n_jobs;
       j += int64_t(gridDim.x) * blockDim.x) {
    const double* xs = x + off[j];
    const double* ys = y + off[j];
    const int n = len[j];
    double r = __longlong_as_double(0x7ff8000000000000ll);   // NaN: pearson raises
    if (n >= 2) {
      Neumaier sx, sy;
      for (int i = 0; i < n; ++i) { sx.add(xs[i]); sy.add(ys[i]); }
      const double dn = small_int_to_double(n);
      const double mx = __ddiv_rn(sx.value(), dn), my = __ddiv_rn(sy.value(), dn);
      Neumaier qx, qy, qxy;
      for (int i = 0; i < n; ++i) {
        const double a = dsub(xs[i], mx), b = dsub(ys[i], my);
        qx.add(dmul(a, a));
        qy.add(dmul(b, b));
      }
      const double sxx = qx.value(), syy = qy.value();
      if (sxx != 0.0 && syy != 0.0) {
        for (int i = 0; i < n; ++i) qxy.add(dmul(dsub(xs[i], mx), dsub(ys[i], my)));
        const double v = __ddiv_rn(qxy.value(), __dsqrt_rn(dmul(sxx, syy)));
        r = fmax(-1.0, fmin(1.0, v));
      }
    }
    rho[j] = r;
    flag[j] = (r == r && fabs(r) > threshold) ? 1 : 0;
  }
}
}  // namespace pdg

using namespace pdg;

extern "C" int pdg_pearson_flags(const double* x, const double* y, const int32_t* off,
                                 const int32_t* len, int64_t n_jobs, double threshold,
                                 double* rho, uint8_t* flag, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && (!x || !y || !off || !len || !rho || !flag))) {
    set_error("pdg_pearson_flags: invalid arguments");
    return PDG_EINVAL;
  }
  if (n_jobs == 0) return PDG_OK;
  int64_t blocks = (n_jobs + 127) / 128;
  const int64_t cap = int64_t(sm_count()) * 16;
  if (blocks > cap) blocks = cap;
  pearson_kernel<<<unsigned(blocks), 128, 0, (cudaStream_t)stream>>>(x, y, off, len, n_jobs,
                                                                    threshold, rho, flag);
  return launch_status("pearson_kernel");
}
