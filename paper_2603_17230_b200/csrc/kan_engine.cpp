// kan_engine.cpp -- host side of the B200 KAN engine behind the C ABI
// (include/kan_b200.h).
//
// Mirrors the reference's model/eval layer (proj/include/kantize/io.hpp:357-386
// model_from_descriptor, layers.hpp:215-308 Model, eval.hpp:83-276
// PreparedModel/model_forward/predict): the descriptor builds the layer stack,
// configure() plays PreparedModel::make once (weights quantized / converted,
// tables built, everything uploaded), forward() runs one fused gather-GEMM
// launch per KAN layer on the caller's stream.  No CPU fallback exists: every
// forward runs on the GPU or returns an error.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/kan_b200.h"
#include "kan_host_math.hpp"
#include "kan_internal.h"
#include "kan_json.hpp"

namespace kan {
// kernels (kan_gemm.cu / kan_fp32.cu)
cudaError_t launch_gather_gemm(bool bf16, int nbp, int mode, const CUtensorMap& xmap,
                               const GemmParams& p, size_t smem, cudaStream_t st);
size_t gemm_smem_bytes(bool bf16, int nbp, int BN, int SA, int SB, int SX, int x_kind,
                       int tab_bytes);
int gemm_ips(bool bf16, int nbp);
int gemm_gs(bool bf16, int nbp);
int gemm_tmem_slots(int BN);
cudaError_t launch_levels(const float* x, int64_t n, const float* thr, float lo, float inv_step,
                          int L, uint16_t* out, cudaStream_t st);
cudaError_t launch_argmax(const float* logits, int64_t M, int N, int ld, int32_t* out,
                          cudaStream_t st);
cudaError_t launch_fp32_layer(const Fp32Params& p, cudaStream_t st);

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LogicError : std::logic_error {
  using std::logic_error::logic_error;
};

static void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t count, bool zero = false) {
    if (count <= n && p) {
      if (zero) ck(cudaMemset(p, 0, count * sizeof(T)), "cudaMemset");
      return;
    }
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    n = count;
    if (zero) ck(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T)), "cudaMemset");
  }
  void upload(const std::vector<T>& v) {
    alloc(v.size());
    if (!v.empty())
      ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy");
  }
};

enum LayerType { L_LINEAR, L_CONV, L_MAXPOOL, L_FLATTEN };

struct Layer {
  LayerType type = L_LINEAR;
  int n_in = 0, n_out = 0;  // linear: features; conv: patch size / c_out
  int c_in = 0, c_out = 0, kernel = 0, stride = 1, padding = 0, window = 2;
  int kan_index = -1;
  std::vector<double> coeffs;  // reference layout [n_in*nb, n_out]
  std::vector<double> base_w;  // [n_in, n_out]
};

// Device-side state of one configured KAN layer.
struct PreparedLayer {
  int layer_index = 0;
  int n_in = 0, N = 0, BN = 0, n_tiles_n = 0, nbp = 8;
  int IPS = 0, GS = 0, n_spline_stages = 0, n_groups = 0, total_stages = 0, silu = 0;
  DevBuf<uint8_t> wt;       // tcgen05 paths: pre-tiled weights
  DevBuf<float> w32, wb32;  // fp32 path
  int Npad = 0;
  // epilogue constants
  int wscheme = 1;
  double f_tensor = 0.0;
  long long z_w = 0;
  DevBuf<double> fs, fb;
  DevBuf<long long> corr_b;
  int b_signed = 1;
};

using EncodeTiledFn = PFN_cuTensorMapEncodeTiled_v12000;

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q),
       "cudaGetDriverEntryPoint");
    if (q != cudaDriverEntryPointSuccess || !ptr) throw CudaError("cuTensorMapEncodeTiled missing");
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// byte offset of 16-byte chunk c of row r in a UMMA K-major SW128 tile
// (matches kan::sw128_off in kan_ptx.cuh)
static inline size_t sw128_off_host(int r, int c) {
  return static_cast<size_t>(r >> 3) * 1024 + static_cast<size_t>(r & 7) * 128 +
         (static_cast<size_t>(c ^ (r & 7)) << 4);
}

static CUtensorMap make_xmap(const void* base, int x_kind, int64_t rows, int cols, int64_t ld,
                             int box_cols) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const size_t esz = x_kind == X_F32 ? 4 : 2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(std::max<int64_t>(rows, 1))};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esz)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), 128u};
  cuuint32_t estr[2] = {1u, 1u};
  // rows of 128 / 64 / 32 bytes are swizzled so the producers' row-per-lane 16-byte
  // reads are bank-conflict free (kan_gemm.cu xtile_off)
  const size_t row_bytes = static_cast<size_t>(box_cols) * esz;
  const CUtensorMapSwizzle sw = row_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = get_encode_fn()(
      &m, x_kind == X_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

}  // namespace kan

using namespace kan;

struct kan_engine {
  int device = 0;
  std::string name;
  Grid grid;
  std::vector<int> input_shape;
  std::vector<Layer> layers;
  int n_kan = 0;
  std::string err;
  // configuration
  bool configured = false;
  kan_config cfg{};
  std::vector<uint8_t> lut;
  Lattice lat;
  std::vector<PreparedLayer> prep;
  DevBuf<float> d_thr;
  DevBuf<uint8_t> d_tab;  // smem table blob (see GemmParams::tab)
  int tab_bytes = 0, off_thr = 0, off_silu = 0;
  double s_s = 1.0;
  int64_t z_s = 0;
  // workspaces
  DevBuf<uint8_t> act[2];
  DevBuf<float> xstage;
  DevBuf<float> logits_tmp;
  DevBuf<uint8_t> io_in, io_out;
  int last_launches = 0;
  // optional per-CTA phase timestamps of each layer's last launch (tuning aid)
  bool timeline = false;
  int dbg_flags = 0;  // KAN_DBG_FLAGS (tuning experiments only)
  std::vector<DevBuf<unsigned long long>> timeline_buf;
  std::vector<int64_t> timeline_ctas;
  // per-layer kernel timing (kan_engine_set_profiling)
  struct PendingTiming {
    int layer;
    cudaEvent_t a, b;
  };
  bool profiling = false;
  std::vector<PendingTiming> pending;
  std::vector<double> layer_ms;
  std::vector<int64_t> layer_count;
  void drain_timings() {
    if (layer_ms.size() < static_cast<size_t>(n_kan)) {
      layer_ms.resize(static_cast<size_t>(n_kan), 0.0);
      layer_count.resize(static_cast<size_t>(n_kan), 0);
    }
    for (auto& t : pending) {
      float ms = 0.f;
      if (cudaEventSynchronize(t.b) == cudaSuccess && cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
        layer_ms[static_cast<size_t>(t.layer)] += ms;
        layer_count[static_cast<size_t>(t.layer)] += 1;
      }
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    pending.clear();
  }
  ~kan_engine() {
    for (auto& t : pending) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
  }

  int64_t input_size() const {
    int64_t n = 1;
    for (int d : input_shape) n *= d;
    return n;
  }
  int output_count() const {
    for (auto it = layers.rbegin(); it != layers.rend(); ++it)
      if (it->type == L_LINEAR || it->type == L_CONV) return it->type == L_LINEAR ? it->n_out : it->c_out;
    throw InvalidArgument("Model::output_count: model has no KAN layers");
  }
  Layer& kan_layer(int i) {
    for (auto& l : layers)
      if (l.kan_index == i) return l;
    throw InvalidArgument("KAN layer index out of range");
  }
};

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

template <class F>
kan_status guarded(kan_engine* e, F&& f) {
  try {
    f();
    if (e) e->err.clear();
    return KAN_OK;
  } catch (const ShapeMismatch& x) {
    if (e) e->err = x.what();
    return KAN_ERR_SHAPE_MISMATCH;
  } catch (const InvalidArgument& x) {
    if (e) e->err = x.what();
    return KAN_ERR_INVALID_ARGUMENT;
  } catch (const FormatError& x) {
    if (e) e->err = x.what();
    return KAN_ERR_FORMAT;
  } catch (const Unsupported& x) {
    if (e) e->err = x.what();
    return KAN_ERR_UNSUPPORTED;
  } catch (const CudaError& x) {
    if (e) e->err = x.what();
    return KAN_ERR_CUDA;
  } catch (const LogicError& x) {
    if (e) e->err = x.what();
    return KAN_ERR_LOGIC;
  } catch (const std::out_of_range& x) {
    if (e) e->err = x.what();
    return KAN_ERR_OUT_OF_RANGE;
  } catch (const std::exception& x) {
    if (e) e->err = x.what();
    return KAN_ERR_INVALID_ARGUMENT;
  }
}

// Model::validate (layers.hpp:252-307)
void validate(kan_engine* e) {
  bool flat = e->input_shape.size() == 1;
  int c = 0, h = 0, w = 0, d = 0;
  if (flat) {
    d = e->input_shape[0];
  } else if (e->input_shape.size() == 3) {
    c = e->input_shape[0];
    h = e->input_shape[1];
    w = e->input_shape[2];
  } else {
    throw ShapeMismatch("Model::validate: input_shape must be [D] or [C,H,W]");
  }
  int idx = 0;
  for (auto& l : e->layers) {
    const std::string si = std::to_string(idx);
    if (l.type == L_LINEAR) {
      if (!flat) throw ShapeMismatch("Model::validate: linear layer " + si + " applied to unflattened tensor");
      if (d != l.n_in)
        throw ShapeMismatch("Model::validate: layer " + si + " expects " + std::to_string(l.n_in) +
                            " inputs, got " + std::to_string(d));
      d = l.n_out;
    } else if (l.type == L_CONV) {
      if (flat) throw ShapeMismatch("Model::validate: conv layer " + si + " applied to flat input");
      if (c != l.c_in)
        throw ShapeMismatch("Model::validate: layer " + si + " expects " + std::to_string(l.c_in) +
                            " channels, got " + std::to_string(c));
      const int sh = h + 2 * l.padding - l.kernel, sw = w + 2 * l.padding - l.kernel;
      if (sh < 0 || sw < 0 || sh % l.stride || sw % l.stride)
        throw ShapeMismatch("Model::validate: layer " + si +
                            " output dimensions are not positive integers for " +
                            std::to_string(h) + "x" + std::to_string(w) + " input");
      c = l.c_out;
      h = sh / l.stride + 1;
      w = sw / l.stride + 1;
    } else if (l.type == L_MAXPOOL) {
      if (flat) throw ShapeMismatch("Model::validate: pool layer on flat input");
      h /= l.window;
      w /= l.window;
    } else {
      if (flat) throw ShapeMismatch("Model::validate: flatten on flat input");
      d = c * h * w;
      flat = true;
    }
    ++idx;
  }
}

// ---- weight preparation ----------------------------------------------------

// per-output-channel symmetric quantization (engine extension; rounding as
// quantize_value's llround, quant.hpp:52)
void quant_per_channel(const std::vector<double>& w, int64_t K, int N, int bits,
                       std::vector<int8_t>& q, std::vector<double>& s) {
  if (bits < 2 || bits > 8) throw InvalidArgument("per-channel weight bits must be in [2,8]");
  const int64_t Q = (int64_t{1} << (bits - 1)) - 1;
  q.assign(static_cast<size_t>(K * N), 0);
  s.assign(static_cast<size_t>(N), 1.0);
  for (int j = 0; j < N; ++j) {
    double mx = 0.0;
    for (int64_t c = 0; c < K; ++c) {
      const double v = std::fabs(w[static_cast<size_t>(c * N + j)]);
      mx = (mx < v) ? v : mx;
    }
    const double sj = (mx > 0.0) ? mx / static_cast<double>(Q) : 1.0;
    s[static_cast<size_t>(j)] = sj;
    for (int64_t c = 0; c < K; ++c) {
      int64_t v = std::llround(w[static_cast<size_t>(c * N + j)] / sj);
      v = v < -Q ? -Q : (v > Q ? Q : v);
      q[static_cast<size_t>(c * N + j)] = static_cast<int8_t>(v);
    }
  }
}

// per-tensor asymmetric quantization, exactly maybe_fake_quant_weights'
// parameters (eval.hpp:70-76 -> RangeCalibrator(widen) + zero_spanning +
// compute_quant_params, quant.hpp:97-125)
// Joint per-output-channel symmetric quantization of spline rows w [K, N] and
// base rows wb [n_in, N] (base values scaled by `ratio` into spline-code
// units): one scale s_j = max(|w[:,j]|, |wb[:,j]*ratio|) / Q per channel.
void quant_joint(const std::vector<double>& w, const std::vector<double>& wb, int64_t K, int n_in,
                 int N, int bits, double ratio, std::vector<int8_t>& q, std::vector<int8_t>& qb,
                 std::vector<double>& s) {
  if (bits < 2 || bits > 8) throw InvalidArgument("per-channel weight bits must be in [2,8]");
  const int64_t Q = (int64_t{1} << (bits - 1)) - 1;
  q.assign(static_cast<size_t>(K * N), 0);
  qb.assign(static_cast<size_t>(n_in) * N, 0);
  s.assign(static_cast<size_t>(N), 1.0);
  auto clampq = [Q](int64_t v) { return static_cast<int8_t>(v < -Q ? -Q : (v > Q ? Q : v)); };
  for (int j = 0; j < N; ++j) {
    double mx = 0.0;
    for (int64_t c = 0; c < K; ++c) {
      const double v = std::fabs(w[static_cast<size_t>(c * N + j)]);
      mx = (mx < v) ? v : mx;
    }
    for (int i = 0; i < n_in; ++i) {
      const double v = std::fabs(wb[static_cast<size_t>(i) * N + j] * ratio);
      mx = (mx < v) ? v : mx;
    }
    const double sj = (mx > 0.0) ? mx / static_cast<double>(Q) : 1.0;
    s[static_cast<size_t>(j)] = sj;
    for (int64_t c = 0; c < K; ++c)
      q[static_cast<size_t>(c * N + j)] = clampq(std::llround(w[static_cast<size_t>(c * N + j)] / sj));
    for (int i = 0; i < n_in; ++i)
      qb[static_cast<size_t>(i) * N + j] =
          clampq(std::llround((wb[static_cast<size_t>(i) * N + j] * ratio) / sj));
  }
}

void quant_per_tensor(const std::vector<double>& w, int bits, std::vector<uint8_t>& q,
                      QParams& qp) {
  if (w.empty()) throw InvalidArgument("empty coefficient matrix");
  double lo = w[0], hi = w[0];
  for (double v : w) {
    lo = (v < lo) ? v : lo;
    hi = (hi < v) ? v : hi;
  }
  if (lo == hi) {
    const double pad = (std::fabs(lo) > 1.0 ? std::fabs(lo) : 1.0) * 2.220446049250313e-16 * 4.0;
    lo -= pad;
    hi += pad;
  }
  lo = (0.0 < lo) ? 0.0 : lo;
  hi = (hi < 0.0) ? 0.0 : hi;
  qp = quant_params(lo, hi, bits);
  q.resize(w.size());
  for (size_t i = 0; i < w.size(); ++i) q[i] = static_cast<uint8_t>(quantize(w[i], qp));
}

// Position of group-input gi inside the SiLU stage's KSTAGE-byte K row; must
// match the producer's shift-register order in kan_gemm.cu.
// Producer thread (row r, K-quarter h) handles inputs [h*IPS/4, (h+1)*IPS/4)
// of every stage and shifts their SiLU codes into a 64-byte register that it
// writes as bytes [64h, 64h+64) of the base stage's row, in stage order.
int silu_pos(bool bf16, int nbp, int gi) {
  const int ips = gemm_ips(bf16, nbp);
  const int q = ips / 4;
  const int s = gi / ips, h = (gi % ips) / q, e = gi % q;
  return h * (bf16 ? 32 : 64) + s * q + e;  // element index in the stage row
}

// byte offset of K byte kb of weight row n in a stage tile: KSTAGE/128 SW128
// blocks of [BN rows][128 B], one per 128 bytes of K
static inline size_t tile_off(int BN, int n, int kb) {
  return static_cast<size_t>(kb >> 7) * BN * 128 + sw128_off_host(n, (kb & 127) >> 4) + (kb & 15);
}

void prepare_gemm_layer(kan_engine* e, const Layer& l, PreparedLayer& pl, bool bf16) {
  const kan_config& cfg = e->cfg;
  const Grid& g = e->grid;
  const int nb = g.nb();
  const int nbp = nb <= 8 ? 8 : 16;
  if (nb > 16) throw Unsupported("G + P > 16 is not supported by the tcgen05 path");
  if (g.P > 3) throw Unsupported("degree > 3 is not supported by the tcgen05 path");
  const int n_in = l.type == L_LINEAR ? l.n_in : l.kernel * l.kernel * l.c_in;
  const int N = l.type == L_LINEAR ? l.n_out : l.c_out;
  pl.n_in = n_in;
  pl.N = N;
  pl.nbp = nbp;
  pl.BN = N > 256 ? 256 : std::max(16, (N + 15) / 16 * 16);
  pl.n_tiles_n = (N + pl.BN - 1) / pl.BN;
  pl.IPS = gemm_ips(bf16, nbp);
  pl.GS = gemm_gs(bf16, nbp);
  pl.silu = cfg.silu_base ? 1 : 0;
  if (pl.silu && l.base_w.size() != static_cast<size_t>(n_in) * N)
    throw InvalidArgument("silu_base requires base weights [n_in, n_out] for every KAN layer");
  pl.n_spline_stages = (n_in + pl.IPS - 1) / pl.IPS;
  pl.n_groups = (pl.n_spline_stages + pl.GS - 1) / pl.GS;
  const int last = pl.n_spline_stages - (pl.n_groups - 1) * pl.GS;
  pl.total_stages = (pl.n_groups - 1) * (pl.GS + pl.silu) + last + pl.silu;
  const int BN = pl.BN;
  const size_t tile_bytes = static_cast<size_t>(BN) * KSTAGE;
  std::vector<uint8_t> wt(static_cast<size_t>(pl.n_tiles_n) * pl.total_stages * tile_bytes, 0);
  const int esz = bf16 ? 2 : 1;

  // element value sources
  std::vector<uint8_t> qw_u8;
  std::vector<int8_t> qw_s8, qwb;
  std::vector<double> s_w, s_wb;
  QParams qpt;
  if (!bf16) {
    pl.wscheme = cfg.w_scheme;
    if (cfg.w_scheme == KAN_W_PER_TENSOR_ASYM) {
      if (pl.silu) throw InvalidArgument("silu_base requires the per-channel weight scheme");
      quant_per_tensor(l.coeffs, cfg.bits_w, qw_u8, qpt);
      pl.b_signed = 0;
    } else if (cfg.w_scheme == KAN_W_PER_CHANNEL_SYM) {
      if (pl.silu) {
        // one scale per output channel over the spline AND base weights, the
        // base weights expressed in spline-code units (ratio = s_s / s_b), so
        // both parts share a single int32 accumulator
        const double ratio = e->s_s / quant_params(0.0, 1.0, cfg.lut_h).scale;
        quant_joint(l.coeffs, l.base_w, static_cast<int64_t>(n_in) * nb, n_in, N, cfg.bits_w,
                    ratio, qw_s8, qwb, s_w);
      } else {
        quant_per_channel(l.coeffs, static_cast<int64_t>(n_in) * nb, N, cfg.bits_w, qw_s8, s_w);
      }
      pl.b_signed = 1;
    } else {
      throw InvalidArgument("unknown weight scheme");
    }
  }
  const int GI = pl.GS * pl.IPS;  // inputs per group
  for (int nt = 0; nt < pl.n_tiles_n; ++nt) {
    for (int grp = 0; grp < pl.n_groups; ++grp) {
      const int nsp = std::min(pl.GS, pl.n_spline_stages - grp * pl.GS);
      for (int s = 0; s < nsp + pl.silu; ++s) {
        const size_t st_idx = static_cast<size_t>(grp) * (pl.GS + pl.silu) + s;
        uint8_t* tile = wt.data() + (static_cast<size_t>(nt) * pl.total_stages + st_idx) * tile_bytes;
        for (int n = 0; n < BN; ++n) {
          const int j = nt * BN + n;
          if (j >= N) continue;
          if (s < nsp) {
            const int i0 = (grp * pl.GS + s) * pl.IPS;
            for (int ii = 0; ii < pl.IPS; ++ii) {
              const int i = i0 + ii;
              if (i >= n_in) break;
              for (int b = 0; b < nb; ++b) {
                const size_t src = (static_cast<size_t>(i) * nb + b) * N + j;
                const int elem = ii * nbp + b;
                const int kb = elem * esz;
                uint8_t* dst = tile + tile_off(BN, n, kb);
                if (bf16) {
                  const __nv_bfloat16 bv = __float2bfloat16_rn(static_cast<float>(l.coeffs[src]));
                  std::memcpy(dst, &bv, 2);
                } else if (pl.b_signed) {
                  dst[0] = static_cast<uint8_t>(qw_s8[src]);
                } else {
                  dst[0] = qw_u8[src];
                }
              }
            }
          } else {
            for (int gi = 0; gi < GI; ++gi) {
              const int i = grp * GI + gi;
              if (i >= n_in) break;
              const int elem = silu_pos(bf16, nbp, gi);
              const int kb = elem * esz;
              uint8_t* dst = tile + tile_off(BN, n, kb);
              const size_t src = static_cast<size_t>(i) * N + j;
              if (bf16) {
                const __nv_bfloat16 bv = __float2bfloat16_rn(static_cast<float>(l.base_w[src]));
                std::memcpy(dst, &bv, 2);
              } else {
                dst[0] = static_cast<uint8_t>(qwb[src]);
              }
            }
          }
        }
      }
    }
  }
  pl.wt.upload(wt);

  if (!bf16) {
    const QParams vq = quant_params(0.0, 1.0, cfg.lut_h);  // s_b = value_qp.scale (lut.hpp:112)
    const double s_b = vq.scale;
    if (pl.wscheme == KAN_W_PER_TENSOR_ASYM) {
      pl.f_tensor = s_b * qpt.scale;
      pl.z_w = qpt.zp;
    } else {
      std::vector<double> fs(static_cast<size_t>(N)), fb(static_cast<size_t>(N), 0.0);
      std::vector<long long> corr(static_cast<size_t>(N), 0);
      for (int j = 0; j < N; ++j) {
        fs[static_cast<size_t>(j)] = s_b * s_w[static_cast<size_t>(j)];
        if (pl.silu) {
          long long cs = 0;
          for (int i = 0; i < n_in; ++i) cs += qwb[static_cast<size_t>(i) * N + j];
          corr[static_cast<size_t>(j)] = e->z_s * cs;
        }
      }
      pl.fs.upload(fs);
      pl.fb.upload(fb);
      pl.corr_b.upload(corr);
    }
  }
}

void prepare_fp32_layer(kan_engine* e, const Layer& l, PreparedLayer& pl) {
  const Grid& g = e->grid;
  const int nb = g.nb();
  if (nb > 16) throw Unsupported("G + P > 16 is not supported");
  if (g.P > 3) throw Unsupported("degree > 3 is not supported");
  const int nbp = nb <= 8 ? 8 : 16;
  const int n_in = l.type == L_LINEAR ? l.n_in : l.kernel * l.kernel * l.c_in;
  const int N = l.type == L_LINEAR ? l.n_out : l.c_out;
  pl.n_in = n_in;
  pl.N = N;
  pl.nbp = nbp;
  pl.Npad = (N + 63) / 64 * 64;
  pl.silu = e->cfg.silu_base ? 1 : 0;
  std::vector<float> w(static_cast<size_t>(n_in) * nbp * pl.Npad, 0.f);
  for (int i = 0; i < n_in; ++i)
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < N; ++j)
        w[(static_cast<size_t>(i) * nbp + b) * pl.Npad + j] =
            static_cast<float>(l.coeffs[(static_cast<size_t>(i) * nb + b) * N + j]);
  pl.w32.upload(w);
  if (pl.silu) {
    if (l.base_w.size() != static_cast<size_t>(n_in) * N)
      throw InvalidArgument("silu_base requires base weights [n_in, n_out] for every KAN layer");
    std::vector<float> wb(static_cast<size_t>(n_in) * pl.Npad, 0.f);
    for (int i = 0; i < n_in; ++i)
      for (int j = 0; j < N; ++j)
        wb[static_cast<size_t>(i) * pl.Npad + j] = static_cast<float>(l.base_w[static_cast<size_t>(i) * N + j]);
    pl.wb32.upload(wb);
  }
}

void configure(kan_engine* e, const kan_config* c) {
  if (!c) throw InvalidArgument("configure: null config");
  DeviceGuard dg(e->device);
  const kan_config cfg = *c;
  if (cfg.mode != KAN_MODE_FP32 && cfg.mode != KAN_MODE_BF16 && cfg.mode != KAN_MODE_BSPLINE_LUT)
    throw InvalidArgument("unknown evaluation mode");
  e->cfg = cfg;
  e->configured = false;
  for (auto& l : e->layers)
    if (l.type == L_CONV) throw Unsupported("conv layers: implicit-im2col path not built yet");
  const Grid& g = e->grid;
  if (cfg.mode == KAN_MODE_BSPLINE_LUT) {
    e->lut = build_lut(g.P, cfg.lut_k, cfg.lut_h);  // validates P, k, h like the reference
    e->lat = Lattice::of(g, cfg.lut_k);
    const int64_t L = e->lat.L;
    const std::vector<float> thr = level_thresholds(g, e->lat);
    e->d_thr.upload(thr);
    std::vector<uint8_t> codes;
    if (cfg.silu_base) {
      std::vector<double> v(static_cast<size_t>(L) + 1);
      double lo = 0.0, hi = 0.0;
      for (int64_t a = 0; a <= L; ++a) {
        const double t = e->lat.dequantize(a);
        v[static_cast<size_t>(a)] = t / (1.0 + std::exp(-t));
        lo = (v[static_cast<size_t>(a)] < lo) ? v[static_cast<size_t>(a)] : lo;
        hi = (hi < v[static_cast<size_t>(a)]) ? v[static_cast<size_t>(a)] : hi;
      }
      const QParams sq = quant_params(lo, hi, 8);
      e->s_s = sq.scale;
      e->z_s = sq.zp;
      codes.resize(static_cast<size_t>(L) + 1);
      for (int64_t a = 0; a <= L; ++a)
        codes[static_cast<size_t>(a)] = static_cast<uint8_t>(quantize(v[static_cast<size_t>(a)], sq));
    }
    // smem table blob: vals[frac] (packed LUT codes per in-interval offset),
    // then the exact level thresholds, then the SiLU codes
    std::vector<uint8_t> blob;
    auto a16 = [](size_t n) { return (n + 15) / 16 * 16; };
    const size_t nfrac = size_t{1} << cfg.lut_k;
    blob.assign(a16(nfrac * 4), 0);
    for (size_t f = 0; f < nfrac; ++f) {
      const uint32_t v = lut_pack(g, cfg.lut_k, e->lut, static_cast<int64_t>(f));  // jj = 0
      std::memcpy(&blob[f * 4], &v, 4);
    }
    e->off_thr = static_cast<int>(blob.size());
    blob.resize(a16(blob.size() + thr.size() * 4), 0);
    std::memcpy(&blob[static_cast<size_t>(e->off_thr)], thr.data(), thr.size() * 4);
    e->off_silu = static_cast<int>(blob.size());
    if (!codes.empty()) {
      blob.insert(blob.end(), codes.begin(), codes.end());
      blob.resize(a16(blob.size()), 0);
    }
    e->tab_bytes = static_cast<int>(blob.size());
    e->d_tab.upload(blob);
    if (cfg.w_scheme == KAN_W_PER_TENSOR_ASYM && (cfg.bits_w < 1 || cfg.bits_w > 8))
      throw InvalidArgument("compute_quant_params: bits must be in [1,8] or 32");
  } else {
    if (cfg.mode == KAN_MODE_FP32 && cfg.out_kind != KAN_OUT_F32)
      throw InvalidArgument("int8 outputs are only produced on the LUT path");
  }
  e->prep.clear();
  e->prep.resize(static_cast<size_t>(e->n_kan));
  e->timeline = std::getenv("KAN_TIMELINE") != nullptr;
  e->dbg_flags = std::getenv("KAN_DBG_FLAGS") ? std::atoi(std::getenv("KAN_DBG_FLAGS")) : 0;
  e->timeline_buf.clear();
  e->timeline_buf.resize(static_cast<size_t>(e->n_kan));
  e->timeline_ctas.assign(static_cast<size_t>(e->n_kan), 0);
  for (auto& l : e->layers) {
    if (l.type != L_LINEAR && l.type != L_CONV) continue;
    const int nb = g.nb();
    const int n_in = l.type == L_LINEAR ? l.n_in : l.kernel * l.kernel * l.c_in;
    const int N = l.type == L_LINEAR ? l.n_out : l.c_out;
    if (l.coeffs.size() != static_cast<size_t>(n_in) * nb * N)
      throw InvalidArgument("coefficients of KAN layer " + std::to_string(l.kan_index) + " not set");
    PreparedLayer& pl = e->prep[static_cast<size_t>(l.kan_index)];
    pl.layer_index = l.kan_index;
    if (cfg.mode == KAN_MODE_FP32)
      prepare_fp32_layer(e, l, pl);
    else
      prepare_gemm_layer(e, l, pl, cfg.mode == KAN_MODE_BF16);
  }
  e->configured = true;
}

// Ring depths for the smem budget: the A ring only decouples producers from
// the MMA (2 slots); the weight and activation rings hide L2 / HBM latency, so
// they get equal depth first and the activation ring takes what is left.
void pick_stages(bool bf16, int nbp, int BN, int x_kind, int tab_bytes, int& SA, int& SB, int& SX) {
  const size_t budget = 232448;
  SA = gemm_tmem_slots(BN);  // the A ring lives in TMEM
  for (SB = 12; SB >= 2; --SB)
    if (gemm_smem_bytes(bf16, nbp, BN, SA, SB, SB, x_kind, tab_bytes) <= budget) break;
  if (SB < 2) throw Unsupported("tile configuration exceeds shared memory");
  for (SX = 24; SX > SB; --SX)
    if (gemm_smem_bytes(bf16, nbp, BN, SA, SB, SX, x_kind, tab_bytes) <= budget) break;
  if (gemm_smem_bytes(bf16, nbp, BN, SA, SB, SX, x_kind, tab_bytes) > budget) SX = SB;
}

struct LayerIO {
  const void* x;
  int x_kind;
  int64_t ld_x;
  void* out;
  int epi;
  int64_t ld_out;
  void* out2;
};

void run_gemm_layer(kan_engine* e, PreparedLayer& pl, int64_t M, const LayerIO& io, cudaStream_t st) {
  const bool bf16 = e->cfg.mode == KAN_MODE_BF16;
  GemmParams p{};
  p.M = static_cast<int>(M);
  p.n_in = pl.n_in;
  p.N = pl.N;
  p.BN = pl.BN;
  p.n_tiles_n = pl.n_tiles_n;
  p.IPS = pl.IPS;
  p.GS = pl.GS;
  p.n_spline_stages = pl.n_spline_stages;
  p.n_groups = pl.n_groups;
  p.silu = pl.silu;
  p.total_stages = pl.total_stages;
  p.x_kind = io.x_kind;
  p.L = bf16 ? 0 : static_cast<int>(e->lat.L);
  p.k = e->lat.k;
  p.tab = e->d_tab.p;
  p.tab_bytes = e->tab_bytes;
  p.off_thr = e->off_thr;
  p.off_silu = e->off_silu;
  p.lo_f = bf16 ? 0.f : static_cast<float>(-e->grid.lo / e->lat.step);
  p.inv_step_f = bf16 ? 0.f : static_cast<float>(1.0 / e->lat.step);
  p.flo = static_cast<float>(e->grid.lo);
  p.fhi_open = std::nextafter(static_cast<float>(e->grid.hi), static_cast<float>(e->grid.lo));
  p.finv_delta = static_cast<float>(1.0 / e->grid.delta);
  p.G = e->grid.G;
  p.P = e->grid.P;
  p.wt = pl.wt.p;
  p.b_signed = pl.b_signed;
  p.m_tiles = static_cast<int>((M + 127) / 128);
  p.dbg = nullptr;
  p.dbg_flags = e->dbg_flags;
  const int tb = bf16 ? 0 : e->tab_bytes;
  int SA = 2, SB = 2, SX = 2;
  pick_stages(bf16, pl.nbp, pl.BN, io.x_kind, tb, SA, SB, SX);
  p.SA = SA;
  p.SB = SB;
  p.SX = SX;
  // split-K over a cluster (2, 4 or 8 CTAs along z) when the tile grid
  // under-fills the 148 SMs; the partial tiles are summed through DSMEM, so
  // they must fit in the idle A/B rings.
  const int tiles = p.m_tiles * p.n_tiles_n;
  const size_t red_bytes = static_cast<size_t>(128) * (pl.BN + 4) * 4;
  const size_t ring_bytes = static_cast<size_t>(SB) * pl.BN * KSTAGE +
                            static_cast<size_t>(SX) * 128 * pl.IPS * (io.x_kind == X_F32 ? 4 : 2);
  int want = e->cfg.split_k > 0 ? e->cfg.split_k : 1;
  if (e->cfg.split_k <= 0 && tiles < 148) want = (148 + tiles - 1) / tiles;
  int splits = 1;
  for (int c : {8, 4, 2})
    if (c <= want && c <= pl.n_groups && red_bytes <= ring_bytes) {
      splits = c;
      break;
    }
  const int gps = (pl.n_groups + splits - 1) / splits;
  p.splits = splits;
  p.groups_per_split = gps;
  if (e->timeline) {
    const size_t n = static_cast<size_t>(splits) * p.m_tiles * p.n_tiles_n * 8;
    auto& buf = e->timeline_buf[static_cast<size_t>(pl.layer_index)];
    buf.alloc(n, true);
    p.dbg = buf.p;
    e->timeline_ctas[static_cast<size_t>(pl.layer_index)] = static_cast<int64_t>(n / 8);
  }
  p.epi = io.epi;
  p.out = io.out;
  p.out2 = io.out2;
  p.ld_out = static_cast<int>(io.ld_out);
  p.f_tensor = pl.f_tensor;
  p.z_w = pl.z_w;
  p.fs = pl.fs.p;
  p.fb = pl.fb.p;
  p.corr_b = pl.corr_b.p;
  p.n_lo = e->grid.lo;
  p.n_hi_open = e->grid.hi_open();
  p.n_step = bf16 ? 1.0 : e->lat.step;
  p.n_inv_step = 1.0 / p.n_step;
  p.n_L = static_cast<int>(e->lat.L);
  p.out_scale = e->cfg.out_scale;
  p.inv_out_scale = 1.0 / e->cfg.out_scale;
  const CUtensorMap xmap = make_xmap(io.x, io.x_kind, M, pl.n_in, io.ld_x, pl.IPS);
  const size_t smem = gemm_smem_bytes(bf16, pl.nbp, pl.BN, SA, SB, SX, io.x_kind, tb);
  // kernel variant: 0 plain, 1 per-tensor zero point (reference scheme), 2 SiLU base
  const int mode = pl.silu ? 2 : ((!bf16 && pl.wscheme == KAN_W_PER_TENSOR_ASYM) ? 1 : 0);
  ck(launch_gather_gemm(bf16, pl.nbp, mode, xmap, p, smem, st), "gather_gemm launch");
  e->last_launches += 1;
}

void run_fp32_layer(kan_engine* e, PreparedLayer& pl, int64_t M, const float* x, int64_t ld_x,
                    float* out, int64_t ld_out, cudaStream_t st) {
  Fp32Params p{};
  p.M = static_cast<int>(M);
  p.n_in = pl.n_in;
  p.N = pl.N;
  p.NBP = pl.nbp;
  p.Npad = pl.Npad;
  p.x = x;
  p.ld_x = static_cast<int>(ld_x);
  p.w = pl.w32.p;
  p.wb = pl.silu ? pl.wb32.p : nullptr;
  p.out = out;
  p.ld_out = static_cast<int>(ld_out);
  p.lo = static_cast<float>(e->grid.lo);
  p.hi_open = std::nextafter(static_cast<float>(e->grid.hi), static_cast<float>(e->grid.lo));
  p.inv_delta = static_cast<float>(1.0 / e->grid.delta);
  p.G = e->grid.G;
  p.P = e->grid.P;
  ck(launch_fp32_layer(p, st), "fp32 layer launch");
  e->last_launches += 1;
}

// round a row pitch (elements) so the byte pitch is a multiple of 16 (TMA)
int64_t pitch16(int64_t n, int esz) {
  const int64_t q = 16 / esz;
  return (n + q - 1) / q * q;
}

void forward(kan_engine* e, const float* x, int64_t M, void* out, cudaStream_t st) {
  if (!e->configured) throw LogicError("forward: engine not configured");
  if (M < 0) throw InvalidArgument("forward: negative batch");
  DeviceGuard dg(e->device);
  e->last_launches = 0;
  if (M == 0) return;
  if (e->input_shape.size() != 1) throw Unsupported("image models: conv path not built yet");
  const int64_t D = e->input_size();
  const bool lut = e->cfg.mode == KAN_MODE_BSPLINE_LUT;
  const bool fp32 = e->cfg.mode == KAN_MODE_FP32;
  // input pitch must be a multiple of 16 bytes for TMA
  const float* xin = x;
  int64_t ldx = D;
  if (!fp32 && (D * 4) % 16 != 0) {
    ldx = pitch16(D, 4);
    e->xstage.alloc(static_cast<size_t>(M * ldx));
    ck(cudaMemcpy2DAsync(e->xstage.p, ldx * 4, x, D * 4, D * 4, M, cudaMemcpyDeviceToDevice, st),
       "stage input");
    xin = e->xstage.p;
  }
  // count KAN layers
  std::vector<const Layer*> kl;
  for (auto& l : e->layers)
    if (l.type == L_LINEAR) kl.push_back(&l);
  const void* cur = xin;
  int cur_kind = X_F32;
  int64_t cur_ld = ldx;
  int pp = 0;
  for (size_t li = 0; li < kl.size(); ++li) {
    const Layer& l = *kl[li];
    PreparedLayer& pl = e->prep[static_cast<size_t>(l.kan_index)];
    const bool last = li + 1 == kl.size();
    LayerIO io{};
    io.x = cur;
    io.x_kind = cur_kind;
    io.ld_x = cur_ld;
    void* dst;
    int64_t ld_out;
    int out_kind;
    if (last) {
      dst = out;
      ld_out = pl.N;
      out_kind = (lut && e->cfg.out_kind == KAN_OUT_I8) ? EPI_I8 : EPI_F32;
    } else {
      const int esz = lut ? 2 : 4;
      ld_out = pitch16(pl.N, esz);
      e->act[pp].alloc(static_cast<size_t>(M * ld_out * esz));
      dst = e->act[pp].p;
      out_kind = lut ? EPI_LEVEL : EPI_F32;
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    unsigned ev_flags = cudaEventRecordDefault;
    if (e->profiling) {
      ck(cudaEventCreate(&ev0), "cudaEventCreate");
      ck(cudaEventCreate(&ev1), "cudaEventCreate");
      // External records become graph nodes under stream capture, so the pair
      // brackets the kernel node itself when the forward is replayed from a graph
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      ck(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
      ev_flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
      ck(cudaEventRecordWithFlags(ev0, st, ev_flags), "cudaEventRecord");
    }
    if (fp32) {
      run_fp32_layer(e, pl, M, static_cast<const float*>(cur), cur_ld, static_cast<float*>(dst),
                     ld_out, st);
    } else {
      io.out = dst;
      io.epi = out_kind;
      io.ld_out = ld_out;
      run_gemm_layer(e, pl, M, io, st);
    }
    if (e->profiling) {
      ck(cudaEventRecordWithFlags(ev1, st, ev_flags), "cudaEventRecord");
      e->pending.push_back({l.kan_index, ev0, ev1});
    }
    cur = dst;
    cur_kind = lut ? X_U16 : X_F32;
    cur_ld = ld_out;
    pp ^= 1;
  }
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

kan_status kan_engine_create(const char* descriptor_json, int device, kan_engine** out) {
  if (!out || !descriptor_json) return KAN_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  auto e = std::make_unique<kan_engine>();
  e->device = device;
  kan_status st = guarded(e.get(), [&] {
    const Json j = Json::parse(descriptor_json);
    double lo = -1.0, hi = 1.0;
    if (j.has("domain")) {
      lo = j.at("domain").at(0).number();
      hi = j.at("domain").at(1).number();
    }
    e->grid = Grid::build(j.at("grid").at("intervals").integer(), j.at("grid").at("degree").integer(), lo, hi);
    if (j.has("name")) e->name = j.at("name").string();
    for (const auto& d : j.at("input").arr) e->input_shape.push_back(d.integer());
    int kan_idx = 0;
    for (const auto& jl : j.at("layers").arr) {
      Layer l;
      const std::string type = jl.at("type").string();
      if (type == "linear") {
        l.type = L_LINEAR;
        l.n_in = jl.at("n_in").integer();
        l.n_out = jl.at("n_out").integer();
        l.kan_index = kan_idx++;
      } else if (type == "conv") {
        l.type = L_CONV;
        l.c_in = jl.at("c_in").integer();
        l.c_out = jl.at("c_out").integer();
        l.kernel = jl.at("kernel").integer();
        l.stride = jl.value_int("stride", 1);
        l.padding = jl.value_int("padding", 0);
        l.n_in = l.kernel * l.kernel * l.c_in;
        l.n_out = l.c_out;
        l.kan_index = kan_idx++;
      } else if (type == "maxpool") {
        l.type = L_MAXPOOL;
        l.window = jl.value_int("window", 2);
      } else if (type == "flatten") {
        l.type = L_FLATTEN;
      } else {
        throw FormatError("model_from_descriptor: unknown layer type '" + type + "'");
      }
      e->layers.push_back(std::move(l));
    }
    e->n_kan = kan_idx;
    validate(e.get());
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw InvalidArgument("no such CUDA device");
  });
  if (st != KAN_OK) {
    // keep the handle so the caller can read the message, then the caller destroys it
    *out = e.release();
    return st;
  }
  *out = e.release();
  return KAN_OK;
}

void kan_engine_destroy(kan_engine* e) {
  if (!e) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(e->device);
  delete e;
  cudaSetDevice(prev);
}

const char* kan_engine_last_error(const kan_engine* e) { return e ? e->err.c_str() : "null engine"; }

int kan_engine_num_kan_layers(const kan_engine* e) { return e ? e->n_kan : 0; }
int64_t kan_engine_input_size(const kan_engine* e) { return e ? e->input_size() : 0; }
int kan_engine_output_count(const kan_engine* e) {
  try {
    return e ? e->output_count() : 0;
  } catch (...) {
    return 0;
  }
}

kan_status kan_engine_layer_shape(const kan_engine* e, int layer, int* n_in, int* n_out) {
  return guarded(const_cast<kan_engine*>(e), [&] {
    if (!e) throw InvalidArgument("null engine");
    Layer& l = const_cast<kan_engine*>(e)->kan_layer(layer);
    if (n_in) *n_in = l.n_in;
    if (n_out) *n_out = l.n_out;
  });
}

kan_status kan_engine_set_coeffs(kan_engine* e, int layer, const double* coeffs, int64_t n,
                                 const double* base_w, int64_t n_base) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    Layer& l = e->kan_layer(layer);
    const int64_t want = static_cast<int64_t>(l.n_in) * e->grid.nb() * l.n_out;
    if (n != want || !coeffs)
      throw ShapeMismatch("set_coeffs: expected " + std::to_string(want) + " coefficients, got " +
                          std::to_string(n));
    l.coeffs.assign(coeffs, coeffs + n);
    if (base_w) {
      if (n_base != static_cast<int64_t>(l.n_in) * l.n_out)
        throw ShapeMismatch("set_coeffs: base weights must be [n_in, n_out]");
      l.base_w.assign(base_w, base_w + n_base);
    } else {
      l.base_w.clear();
    }
    e->configured = false;
  });
}

kan_status kan_engine_configure(kan_engine* e, const kan_config* cfg) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] { configure(e, cfg); });
}

kan_status kan_engine_forward(kan_engine* e, const float* x_dev, int64_t batch, void* out_dev,
                              void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (batch > 0 && (!x_dev || !out_dev)) throw InvalidArgument("forward: null buffer");
    forward(e, x_dev, batch, out_dev, static_cast<cudaStream_t>(stream));
  });
}

kan_status kan_engine_forward_host(kan_engine* e, const float* x_host, int64_t batch,
                                   void* out_host, void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (!e->configured) throw LogicError("forward: engine not configured");
    DeviceGuard dg(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t D = e->input_size();
    const size_t ob = static_cast<size_t>(batch) * e->output_count() *
                      ((e->cfg.mode == KAN_MODE_BSPLINE_LUT && e->cfg.out_kind == KAN_OUT_I8) ? 1 : 4);
    e->io_in.alloc(static_cast<size_t>(batch * D) * 4);
    e->io_out.alloc(ob);
    if (batch > 0)
      ck(cudaMemcpyAsync(e->io_in.p, x_host, static_cast<size_t>(batch * D) * 4,
                         cudaMemcpyHostToDevice, st),
         "H2D");
    forward(e, reinterpret_cast<const float*>(e->io_in.p), batch, e->io_out.p, st);
    if (batch > 0) ck(cudaMemcpyAsync(out_host, e->io_out.p, ob, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "stream sync");
  });
}

kan_status kan_engine_predict(kan_engine* e, const float* x_dev, int64_t batch,
                              int32_t* labels_dev, void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (!e->configured) throw LogicError("predict: engine not configured");
    if (e->cfg.out_kind != KAN_OUT_F32) throw InvalidArgument("predict needs fp32 logits");
    DeviceGuard dg(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int N = e->output_count();
    e->logits_tmp.alloc(static_cast<size_t>(batch) * N);
    forward(e, x_dev, batch, e->logits_tmp.p, st);
    const int launches = e->last_launches;
    ck(launch_argmax(e->logits_tmp.p, batch, N, N, labels_dev, st), "argmax");
    e->last_launches = launches + (batch > 0 ? 1 : 0);
  });
}

kan_status kan_engine_layer_levels(kan_engine* e, int layer, const float* x_dev, int64_t n,
                                   uint16_t* levels_dev, void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (!e->configured || e->cfg.mode != KAN_MODE_BSPLINE_LUT)
      throw LogicError("layer_levels: engine not configured for bspline-lut");
    (void)e->kan_layer(layer);  // one grid per model (Model::grid, layers.hpp:224-230)
    DeviceGuard dg(e->device);
    e->last_launches = 0;
    if (n == 0) return;
    ck(launch_levels(x_dev, n, e->d_thr.p, static_cast<float>(e->grid.lo),
                     static_cast<float>(1.0 / e->lat.step), static_cast<int>(e->lat.L), levels_dev,
                     static_cast<cudaStream_t>(stream)),
       "levels launch");
    e->last_launches = 1;
  });
}

kan_status kan_engine_layer_accumulators(kan_engine* e, int layer, const uint16_t* levels_dev,
                                         int64_t batch, int32_t* acc_s_dev, int32_t* acc_b_dev,
                                         void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (!e->configured || e->cfg.mode != KAN_MODE_BSPLINE_LUT)
      throw LogicError("layer_accumulators: engine not configured for bspline-lut");
    Layer& l = e->kan_layer(layer);
    if (l.type != L_LINEAR) throw Unsupported("layer_accumulators: linear layers only");
    DeviceGuard dg(e->device);
    e->last_launches = 0;
    if (batch == 0) return;
    PreparedLayer& pl = e->prep[static_cast<size_t>(layer)];
    const int64_t ld = pitch16(pl.n_in, 2);
    const uint16_t* src = levels_dev;
    if (ld != pl.n_in) {
      e->xstage.alloc(static_cast<size_t>(batch * ld + 1) / 2 + 1);
      ck(cudaMemcpy2DAsync(e->xstage.p, ld * 2, levels_dev, pl.n_in * 2, pl.n_in * 2, batch,
                           cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)),
         "stage levels");
      src = reinterpret_cast<const uint16_t*>(e->xstage.p);
    }
    LayerIO io{};
    io.x = src;
    io.x_kind = X_U16;
    io.ld_x = ld;
    io.out = acc_s_dev;
    io.out2 = acc_b_dev;
    io.epi = EPI_RAW;
    io.ld_out = pl.N;
    run_gemm_layer(e, pl, batch, io, static_cast<cudaStream_t>(stream));
  });
}

int64_t kan_engine_lut(const kan_engine* e, uint8_t* out, int64_t cap) {
  if (!e || !e->configured || e->lut.empty()) return 0;
  const int64_t n = static_cast<int64_t>(e->lut.size());
  if (out && cap >= n) std::memcpy(out, e->lut.data(), static_cast<size_t>(n));
  return n;
}

int kan_engine_last_launches(const kan_engine* e) { return e ? e->last_launches : 0; }

int64_t kan_engine_layer_timeline(kan_engine* e, int layer, unsigned long long* out, int64_t cap) {
  if (!e || layer < 0 || layer >= static_cast<int>(e->timeline_ctas.size())) return 0;
  const int64_t n = e->timeline_ctas[static_cast<size_t>(layer)] * 8;
  if (out && cap >= n && n > 0) {
    DeviceGuard dg(e->device);
    cudaDeviceSynchronize();
    cudaMemcpy(out, e->timeline_buf[static_cast<size_t>(layer)].p, static_cast<size_t>(n) * 8,
               cudaMemcpyDeviceToHost);
  }
  return n;
}

kan_status kan_engine_set_profiling(kan_engine* e, int on) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    DeviceGuard dg(e->device);
    e->drain_timings();
    e->layer_ms.assign(static_cast<size_t>(e->n_kan), 0.0);
    e->layer_count.assign(static_cast<size_t>(e->n_kan), 0);
    e->profiling = on != 0;
  });
}

kan_status kan_engine_layer_time_ms(kan_engine* e, int layer, double* total_ms, int64_t* count) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (layer < 0 || layer >= e->n_kan) throw InvalidArgument("KAN layer index out of range");
    DeviceGuard dg(e->device);
    e->drain_timings();
    if (total_ms) *total_ms = e->layer_ms[static_cast<size_t>(layer)];
    if (count) *count = e->layer_count[static_cast<size_t>(layer)];
  });
}

int64_t kan_lut_build(int degree, int k, int h, uint8_t* out, int64_t cap) {
  try {
    const auto lut = build_lut(degree, k, h);
    const int64_t n = static_cast<int64_t>(lut.size());
    if (out && cap >= n) std::memcpy(out, lut.data(), static_cast<size_t>(n));
    return n;
  } catch (...) {
    return -KAN_ERR_INVALID_ARGUMENT;
  }
}

int64_t kan_lattice_thresholds(int intervals, int degree, double lo, double hi, int k, float* out,
                               int64_t cap) {
  try {
    const Grid g = Grid::build(intervals, degree, lo, hi);
    const auto thr = level_thresholds(g, Lattice::of(g, k));
    const int64_t n = static_cast<int64_t>(thr.size());
    if (out && cap >= n) std::memcpy(out, thr.data(), static_cast<size_t>(n) * sizeof(float));
    return n;
  } catch (...) {
    return -KAN_ERR_INVALID_ARGUMENT;
  }
}

}  // extern "C"
