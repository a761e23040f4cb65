// Exact-order nest evaluator: the B200 replacement of the reference's
// per-point interpreter (pkg/src/tendist/cin.py:420-477, _run_leaf :399-417,
// resolve_var :307-330).
//
// Any leaf statement over any scheduled loop nest runs here with the
// reference's accumulation order: loops that determine the output coordinate
// ("parallel" loops) become GPU threads, and each thread walks the remaining
// loops lexicographically in nest order, doing out += value per point exactly
// as the interpreter does.  Divide/split guards skip phantom points, rotate
// offsets wrap modulo the extent.  If the output coordinate is not an
// injective function of the parallel loops the host sets `serial` and one
// thread walks the whole nest.  This is the path for arbitrary statements and
// for bitwise parity runs; the hot leaves have dedicated kernels.
#include "common.cuh"
#include "interp.cuh"

namespace td {

struct NestState {
  int64_t lv[TD_MAX_LOOPS];
  int64_t val[TD_MAX_VARS];
};

// resolve every slot; false if some slot is phantom and needed
__device__ __forceinline__ bool resolve(const td_nest_prog& p, NestState& s, bool* ph) {
  for (int v = 0; v < p.nvars; ++v) {
    const td_var_def& d = p.vars[v];
    bool phantom = false;
    int64_t x = 0;
    if (d.kind == TD_VAR_LOOP) {
      x = s.lv[d.a];
    } else if (d.kind == TD_VAR_STRIP) {
      phantom = ph[d.a] || ph[d.b];
      x = s.val[d.a] * d.block + s.val[d.b];
      if (x >= d.extent) phantom = true;
    } else {
      phantom = ph[d.a];
      x = s.val[d.a];
      for (int o = 0; o < d.nover; ++o) {
        phantom |= ph[d.over[o]];
        x += s.val[d.over[o]];
      }
      x %= d.extent;
    }
    s.val[v] = x;
    ph[v] = phantom;
  }
  return true;
}

__device__ __forceinline__ bool access_ok(const td_access& a, const bool* ph) {
  for (int d = 0; d < a.ndim; ++d)
    if (ph[a.slot[d]]) return false;
  return true;
}

__device__ __forceinline__ const double* address(const td_access& a, const NestState& s) {
  int64_t off = 0;
  for (int d = 0; d < a.ndim; ++d) off += (s.val[a.slot[d]] - a.origin[d]) * a.stride[d];
  return a.base + off;
}

__device__ __forceinline__ double eval(const td_nest_prog& p, const NestState& s) {
  double st[16];
  int sp = 0;
  for (int c = 0; c < p.ncode; ++c) {
    const int op = p.op[c];
    if (op == TD_OP_CONST) st[sp++] = p.konst[c];
    else if (op == TD_OP_LOAD) st[sp++] = *address(p.acc[p.arg[c]], s);
    else if (op == TD_OP_ADD) { --sp; st[sp - 1] = st[sp - 1] + st[sp]; }
    else { --sp; st[sp - 1] = st[sp - 1] * st[sp]; }
  }
  return st[0];
}

// a point is live when every variable used by some access resolved non-phantom
__device__ __forceinline__ bool point_live(const td_nest_prog& p, const bool* ph) {
  if (!access_ok(p.out, ph)) return false;
  for (int a = 0; a < p.nacc; ++a)
    if (!access_ok(p.acc[a], ph)) return false;
  return true;
}

__global__ void nest_kernel(const __grid_constant__ td_nest_prog p, int64_t npoints) {
  bool is_par[TD_MAX_LOOPS];
  for (int l = 0; l < p.nloops; ++l) is_par[l] = false;
  for (int q = 0; q < p.npar; ++q) is_par[p.par[q]] = true;

  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < npoints;
       t += int64_t(gridDim.x) * blockDim.x) {
    NestState s;
    bool ph[TD_MAX_VARS];
    // decode the parallel loops (row-major in nest order)
    int64_t rem = t;
    for (int q = p.npar - 1; q >= 0; --q) {
      const int l = p.par[q];
      const int64_t ext = p.hi[l] - p.lo[l];
      s.lv[l] = p.lo[l] + rem % ext;
      rem /= ext;
    }
    // sequential odometer over the other loops, lexicographic in nest order
    bool empty = false;
    for (int l = 0; l < p.nloops; ++l)
      if (!is_par[l]) {
        s.lv[l] = p.lo[l];
        if (p.hi[l] <= p.lo[l]) empty = true;
      }
    double* outp = nullptr;
    double accv = 0.0;
    bool have = false;
    while (!empty) {
      resolve(p, s, ph);
      if (point_live(p, ph)) {
        double* o = const_cast<double*>(address(p.out, s));
        if (p.serial) {
          const double v = eval(p, s);
          *o = p.reduce ? *o + v : v;
        } else {
          if (!have) {
            outp = o;
            accv = *o;
            have = true;
          }
          const double v = eval(p, s);
          accv = p.reduce ? accv + v : v;
        }
      }
      // advance
      int l = p.nloops - 1;
      for (; l >= 0; --l) {
        if (is_par[l]) continue;
        if (++s.lv[l] < p.hi[l]) break;
        s.lv[l] = p.lo[l];
      }
      if (l < 0) break;
    }
    if (have) *outp = accv;
  }
}

}  // namespace td

extern "C" int td_nest_eval(void* stream, const void* prog, int64_t bytes) {
  using namespace td;
  StreamDevice sd(stream);
  TD_REQUIRE(bytes == (int64_t)sizeof(td_nest_prog), "nest_eval: program is %lld bytes, expected %lld",
             (long long)bytes, (long long)sizeof(td_nest_prog));
  const td_nest_prog& p = *static_cast<const td_nest_prog*>(prog);
  TD_REQUIRE(p.nloops >= 0 && p.nloops <= TD_MAX_LOOPS && p.nvars <= TD_MAX_VARS && p.nacc <= TD_MAX_ACC &&
                 p.ncode >= 1 && p.ncode <= TD_MAX_CODE,
             "nest_eval: program limits exceeded");
  int64_t npoints = 1;
  if (!p.serial) {
    for (int q = 0; q < p.npar; ++q) {
      const int64_t ext = p.hi[p.par[q]] - p.lo[p.par[q]];
      if (ext <= 0) return TD_OK;
      npoints *= ext;
    }
  }
  const int threads = p.serial ? 1 : 128;
  const int64_t blocks = p.serial ? 1 : std::max<int64_t>(1, std::min<int64_t>(ceil_div(npoints, threads), 148 * 64));
  nest_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(p, npoints);
  return check_launch("nest_kernel");
}
