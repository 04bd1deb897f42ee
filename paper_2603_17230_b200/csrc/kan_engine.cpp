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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
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
                       int tab_bytes, bool silu, int fused_bytes);
int gemm_ips(bool bf16, int nbp);
int gemm_gs(bool bf16, int nbp);
int gemm_tmem_slots(int BN, int nacc);
int gemm_tmem_accs(int BN, int splits);
cudaError_t launch_levels(const float* x, int64_t n, const float* thr, float nlo_step, float inv_step,
                          int L, uint16_t* out, cudaStream_t st);
cudaError_t launch_argmax(const float* logits, int64_t M, int N, int ld, int32_t* out,
                          cudaStream_t st);
cudaError_t launch_fp32_layer(const Fp32Params& p, cudaStream_t st);
cudaError_t launch_im2col_f32(const float* in, int64_t n_img, int C, int H, int W, int K, int stride, int pad, int Ho,
                              int Wo, float* out, cudaStream_t st);
cudaError_t launch_rows_to_nchw(const float* rows, int64_t n_img, int HW, int N, float* out, cudaStream_t st);
cudaError_t launch_maxpool_f32(const float* in, int64_t planes, int H, int W, int win, float* out, cudaStream_t st);
cudaError_t launch_small_layer(const SmallParams& p, cudaStream_t st);
cudaError_t launch_rows_to_levels(const float* x, int64_t M, int n, int ld_x, uint16_t* out, int ld_o,
                                  const float* thr, float nlo_step, float inv_step, int L, cudaStream_t st);
cudaError_t launch_conv3(int mode, const CUtensorMap& xmap, const GemmParams& p, size_t smem, cudaStream_t st);
size_t conv3_smem_bytes(int BN, int R, int SA, int SB, int SX, int x_kind, int tab_bytes, bool silu);
cudaError_t launch_convw(int mode, const CUtensorMap& xmap, const GemmParams& p, size_t smem, cudaStream_t st);
size_t convw_smem_bytes(int BN, int WR, int CX, int SA, int SB, int SX, int tab_bytes, bool zp, bool silu);
int convw_max_rows();
bool convw_dual_capable(int mode, int epi, int g_img);
size_t small_smem_bytes(const SmallParams& p);
cudaError_t launch_im2col_levels(const float* x, int64_t n_img, int C, int H, int W, int K, int stride, int pad,
                                 int Ho, int Wo, uint16_t* out, int ld_o, const float* thr, float nlo_step,
                                 float inv_step, int L, int lvl0, cudaStream_t st);
cudaError_t launch_nchw_to_nhwc(bool levels, const float* in, int64_t n_img, int C, int HW,
                                void* out, int ldc, const float* thr, float lo, float inv_step,
                                int L, cudaStream_t st);
cudaError_t launch_maxpool(bool levels, const void* in, int64_t n_img, int H, int W, int C,
                           int ld_in, int win, void* out, int ld_out, cudaStream_t st);
cudaError_t launch_avgpool(const void* in, int64_t n_img, int HW, int C, int ld_in, void* out,
                           int ld_out, cudaStream_t st);
// training backward (kan_backward.cu)
struct BwParams {
  int64_t M;
  int n_in, n_out, G, P;
  const float* x;
  int64_t ld_x;
  const float* dy;
  const float* w;
  float* dcoeffs;
  float* dinputs;
  float lo, hi_open, inv_delta;
};
cudaError_t launch_linear_backward(const BwParams& p, cudaStream_t st);
cudaError_t launch_sgd_step(double* w, double* v, const float* g, float* w_bw, float* w32, long long n, int nb,
                            int nbp, int N, int Npad, double lr, double momentum, cudaStream_t st);
cudaError_t launch_softmax_ce(const float* logits, const int32_t* labels, int64_t M, int n, float* loss_rows,
                              float* dlogits, cudaStream_t st);
cudaError_t launch_nchw_to_rows(const float* in, int64_t n_img, int HW, int N, float* rows, cudaStream_t st);
cudaError_t launch_col2im(const float* dpatch, int64_t n_img, int C, int H, int W, int K, int stride, int pad, int Ho,
                          int Wo, float* din, cudaStream_t st);
cudaError_t launch_maxpool_bw(const float* in, int64_t planes, int H, int W, int win, const float* dout, float* din,
                              cudaStream_t st);
// spline-table mode (kan_spline_table.cu)
cudaError_t launch_st_sample(const double* basis, const double* coeffs, int n_in, int n_out, int nb, int Lv,
                             int pass, unsigned long long* mm, uint8_t* T, int Np, double s, double zd,
                             long long qhi, cudaStream_t st);
cudaError_t launch_st_layer(const StParams& p, cudaStream_t st);
size_t st_layer_smem(const StParams& p);
cudaError_t launch_st_levels(const float* x, int64_t n, const float* thr, float inv_s, float zf, int qhi,
                             void* out, int out_u16, cudaStream_t st);
cudaError_t launch_u16_to_u8(const uint16_t* in, int64_t n, uint8_t* out, cudaStream_t st);
cudaError_t launch_count_equal(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* count,
                               cudaStream_t st);
cudaError_t launch_st_maxpool(const uint8_t* in, int64_t planes, int H, int W, int win, uint8_t* out,
                              cudaStream_t st);

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

enum LayerType { L_LINEAR, L_CONV, L_MAXPOOL, L_FLATTEN, L_AVGPOOL };

// Per-sample tensor shape (Model::validate's bookkeeping, layers.hpp:252-307).
// `hw`/`fc` record, for a flat tensor made by flattening an image tensor that
// a layer produced (stored NHWC), its H*W and C: the consuming linear layer
// permutes its coefficient rows from the reference's channel-major order.
struct Shape {
  bool flat = true;
  int c = 0, h = 0, w = 0, d = 0;
  int hw = 0, fc = 0;
  bool operator==(const Shape& o) const {
    return flat == o.flat && (flat ? d == o.d : (c == o.c && h == o.h && w == o.w));
  }
};

struct Layer {
  LayerType type = L_LINEAR;
  int n_in = 0, n_out = 0;  // linear: features; conv: patch size / c_out
  int c_in = 0, c_out = 0, kernel = 0, stride = 1, padding = 0, window = 2;
  int kan_index = -1;
  // engine descriptor extension (additive): named tensors for residual blocks
  std::string id, input_from, residual;
  int src = -1;      // layer whose output feeds this layer (-1: model input)
  int res_src = -2;  // layer whose output is added before re-quantization (-2: none)
  Shape in, out;
  // LUT path storage of this layer's output: fp32 values when some consumer
  // needs values (a residual add, average pooling), else exact lattice levels
  bool store_f32 = false;
  // LUT path: a conv on the model input with fewer channels than one IPS chunk
  // (the ResKAN stem, c_in = 3) runs as a dense GEMM over an explicit level
  // im2col of the NCHW input (c_in*k*k inputs instead of k*k padded chunks)
  bool im2col = false;
  std::vector<double> coeffs;  // reference layout [n_in*nb, n_out]
  std::vector<double> base_w;  // [n_in, n_out]
  // fp32 copy of coeffs for the training backward (uploaded on first use after
  // set_coeffs)
  std::shared_ptr<DevBuf<float>> w_bw;
  // training: fp64 master coefficients and momentum on the device
  // (kan_engine_sgd_step); `coeffs` is stale while master_ahead is set
  std::shared_ptr<DevBuf<double>> w_master, w_vel;
  bool master_ahead = false;
  // spline-table mode: tables supplied by the caller (EvalOptions::tables,
  // eval.hpp:41; e.g. loaded from a .kant container) instead of built from
  // the coefficients; values in the reference layout [n_in][n_out][2^bits_a]
  std::vector<uint8_t> st_values;
  int st_bits_a = 0, st_h = 0;
  double st_qd[2] = {0, 0};
  int64_t st_qi[4] = {0, 0, 0, 0};
};

// Device state of one spline-table layer (SplineTableSet, spline_table.hpp:19-34)
struct StLayer {
  DevBuf<uint8_t> T;  // [roundup4(n_in)][Lv][Np]
  DevBuf<int> vthr;   // next-layer level thresholds on the integer sums (StParams::vthr)
  int n_in = 0, n_out = 0, Np = 0, lpr = 1, col_tiles = 1;
  int bits_a = 0, h = 0;
  double in_s = 1.0, out_s = 1.0;
  int64_t in_z = 0, in_qhi = 0, out_z = 0, out_qhi = 0;
  bool ft = false;  // fake-quant mode: fp32 tables, Np = row bytes (4 per column)
  QParams aq;         // this layer's input quantizer (a_params_for, eval.hpp:55-68)
  DevBuf<float> athr; // its exact fp32 thresholds (empty: the engine-wide st_thr)
};

// Device-side state of one configured KAN layer.
struct PreparedLayer {
  int layer_index = 0;
  int64_t acc_bound = 0;  // worst-case |int32 accumulator| (configure's headroom check)
  int n_in = 0, N = 0, BN = 0, n_tiles_n = 0, nbp = 8;
  int cps = 0;  // conv: IPS-wide channel chunks per tap
  // small-N CUDA-core path (LUT, NBP = 8, N <= 16, per-channel weights)
  bool small = false;
  int n_in8 = 0;
  DevBuf<unsigned long long> swq;  // [n_in][N] 8 basis weights per (input, output)
  DevBuf<int8_t> swqb;             // [N][n_in8] SiLU base weights
  DevBuf<int8_t> swqb_plain;       // [N][n_in] SiLU base weights (fused tail layer), padded to 16 B
  // ky-shared 3x3 conv kernel: weights as [n_tile][(kx, chunk)][ky] tap slots
  // of b_slot3 bytes (SW128 codes part + SW32 SiLU part)
  bool conv3 = false;
  int b_slot3 = 0;
  DevBuf<uint8_t> wt3;
  // window-shared 3x3 conv kernel (kan_convw.cuh): weights as
  // [n_tile][K block of 4 channels][9 taps][BNw rows][32 B] (SW32 K-major)
  bool convw = false;
  bool kymw = false;  // weights laid out for the ky-merged MMA issue
  int bnw = 0, trw = 0, ntw = 0, b_slotw = 0;
  DevBuf<uint8_t> wtw;
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
  bool conv_floor = false;  // descriptor "conv_output": "floor"
  bool input_f32 = false;   // the NHWC copy of the model input keeps fp32 values
  int n_kan = 0;
  std::string err;
  // configuration
  bool configured = false;
  kan_config cfg{};
  std::vector<uint8_t> lut;
  Lattice lat;
  std::vector<PreparedLayer> prep;
  DevBuf<float> d_thr;
  // smem table blobs (see GemmParams::tab): [0] shared tables, [1] lane-
  // private copies (NBP = 8 only; used where shared memory allows)
  struct TabSet {
    DevBuf<uint8_t> buf;
    int bytes = 0, off_thr = 0, off_silu = 0, off_c64 = 0;
  } tabs[3];
  double s_s = 1.0;
  int64_t z_s = 0;
  // workspaces: activation buffer slot of each layer's stored output (-1:
  // none -- views, the last layer, or the model input); slots are reused
  // once every consumer of their tensor has run
  std::vector<int> slot_of;
  struct Slot {
    DevBuf<uint8_t> main;
    DevBuf<uint16_t> lv;  // levels sidecar of an fp32-stored tensor
  };
  std::vector<Slot> slots;
  DevBuf<float> xstage;
  DevBuf<uint8_t> xnhwc;  // NHWC copy of an image model's input
  DevBuf<uint16_t> xlev;  // level prepass of a large fp32-input dense layer
  DevBuf<uint16_t> xcol;  // level im2col of the model input (stem convs)
  DevBuf<float> logits_tmp;
  DevBuf<float> fp_col, fp_rows;  // fp32 conv models: patch rows, layer output rows
  DevBuf<float> bw_drows, bw_dpatch;  // conv backward: dY rows, patch gradients
  // LUT entries read from a .kant container (kan_engine_load): configure uses
  // them when lut_k / lut_h match (EvalOptions::lut, eval.hpp:40)
  std::vector<uint8_t> c_lut;
  int c_lut_k = 0, c_lut_h = 0;
  // fake-quant calibrated activation ranges, one (lo, hi) per KAN layer
  // (EvalOptions::a_ranges, eval.hpp:43-44); empty: the grid bounds
  std::vector<std::pair<double, double>> a_ranges;
  // spline-table mode
  std::vector<StLayer> st;
  QParams st_in;            // input quantizer on the grid bounds (spline_table.hpp:51)
  DevBuf<float> st_thr;     // its exact fp32 thresholds
  DevBuf<uint8_t> st_xlev;  // u8 levels of the model input (image models; dense prepass)
  bool st_prepass = true;   // KAN_ST_PREPASS=0: quantize fp32 rows inside the gather kernel
  DevBuf<uint8_t> st_probe;
  DevBuf<int32_t> pred_tmp;
  DevBuf<unsigned long long> count_tmp;
  DevBuf<uint8_t> io_in, io_out;
  int last_launches = 0;
  // optional per-CTA phase timestamps of each layer's last launch (tuning aid)
  bool timeline = false;
  int dbg_flags = 0;  // KAN_DBG_FLAGS (tuning experiments only)
  int force_tab = -1;  // KAN_TABLES=0/1/2 forces the table variant (tuning only)
  bool epi_stage = true;  // KAN_EPI_STAGE=0 disables the staged fp32 epilogue (tuning only)
  // fp32-input dense layers with at least this many activations get the level
  // prepass (KAN_LEVEL_PREPASS_MIN; tests lower it to exercise the path)
  int64_t prepass_min = std::numeric_limits<int64_t>::max();
  int conv3_mc = 2;  // conv3: CTAs per weight-multicast cluster (KAN_CONV3_MC)
  bool lv_sidecar = true;  // KAN_OPT_LV_SIDECAR=0 disables the levels sidecar (tuning)
  // tuning / debug switches (kan_engine_set_option); configure copies them
  // into the fields above, so nothing is read from the environment
  struct Options {
    bool no_convw = false;
    int convw_rings = 0, convw_tr = 0, convw_mc = 0, convw_bn = 0, convw_lock = 0, convw_dual = 0;
    bool no_fuse = false, fuse_persistent = false, no_kym = false;
    bool no_conv3 = false, no_im2col = false, epi_stage = true, lv_sidecar = true, st_prepass = true;
    bool timeline = false, force_nacc1 = false, record_plan = false;
    int force_bn = 0, tables = -1, conv3_mc = 2, st_slices = 0, dbg_flags = 0;
    int64_t level_prepass_min = std::numeric_limits<int64_t>::max();
  } opt;
  // launch plan of the last forward (opt.record_plan): one line per kernel
  std::string plan;
  void plan_add(const char* kernel, int layer, int epi, int res, int lv, int N, int BN, int splits, int mode,
                const char* extra = "") {
    char buf[200];
    std::snprintf(buf, sizeof(buf), "%s layer=%d epi=%d res=%d lv=%d N=%d BN=%d splits=%d mode=%d%s\n", kernel, layer,
                  epi, res, lv, N, BN, splits, mode, extra);
    plan += buf;
  }
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
  // sharded forward (kan_engine_forward_sharded): this engine's own stream and
  // completion event, and a staging buffer for logits that cannot be written
  // in place (another device, or a misaligned shard offset)
  cudaStream_t own_stream = nullptr;
  cudaEvent_t shard_done = nullptr;
  DevBuf<uint8_t> shard_out;
  cudaStream_t stream_own() {
    if (!own_stream) ck(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking), "stream create");
    return own_stream;
  }
  cudaEvent_t done_event() {
    if (!shard_done) ck(cudaEventCreateWithFlags(&shard_done, cudaEventDisableTiming), "event create");
    return shard_done;
  }
  ~kan_engine() {
    for (auto& t : pending) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    if (own_stream) cudaStreamDestroy(own_stream);
    if (shard_done) cudaEventDestroy(shard_done);
  }

  int64_t input_size() const {
    int64_t n = 1;
    for (int d : input_shape) n *= d;
    return n;
  }
  // values per sample of the model output (the last layer's tensor, flattened)
  int output_count() const {
    if (layers.empty()) throw InvalidArgument("Model::output_count: model has no layers");
    const Shape& o = layers.back().out;
    return o.flat ? o.d : o.c * o.h * o.w;
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

// Model::validate (layers.hpp:252-307), extended additively with named
// tensors (id / input_from / residual) and global average pooling.
void validate(kan_engine* e) {
  Shape cur;
  if (e->input_shape.size() == 1) {
    cur.d = e->input_shape[0];
  } else if (e->input_shape.size() == 3) {
    cur.flat = false;
    cur.c = e->input_shape[0];
    cur.h = e->input_shape[1];
    cur.w = e->input_shape[2];
  } else {
    throw ShapeMismatch("Model::validate: input_shape must be [D] or [C,H,W]");
  }
  struct Named {
    int layer;
    Shape shape;
  };
  std::vector<std::pair<std::string, Named>> named{{"input", {-1, cur}}};
  auto find = [&](const std::string& n, const std::string& si) -> const Named& {
    for (auto& kv : named)
      if (kv.first == n) return kv.second;
    throw FormatError("model_from_descriptor: layer " + si + " refers to unknown tensor '" + n + "'");
  };
  int idx = 0, prev = -1;
  for (auto& l : e->layers) {
    const std::string si = std::to_string(idx);
    Shape s = cur;
    l.src = prev;
    if (!l.input_from.empty()) {
      const Named& nm = find(l.input_from, si);
      s = nm.shape;
      l.src = nm.layer;
    }
    l.in = s;
    Shape o;
    if (l.type == L_LINEAR) {
      if (!s.flat) throw ShapeMismatch("Model::validate: linear layer " + si + " applied to unflattened tensor");
      if (s.d != l.n_in)
        throw ShapeMismatch("Model::validate: layer " + si + " expects " + std::to_string(l.n_in) +
                            " inputs, got " + std::to_string(s.d));
      o.d = l.n_out;
    } else if (l.type == L_CONV) {
      if (s.flat) throw ShapeMismatch("Model::validate: conv layer " + si + " applied to flat input");
      if (s.c != l.c_in)
        throw ShapeMismatch("Model::validate: layer " + si + " expects " + std::to_string(l.c_in) +
                            " channels, got " + std::to_string(s.c));
      const int sh = s.h + 2 * l.padding - l.kernel, sw = s.w + 2 * l.padding - l.kernel;
      // the reference requires the stride to divide the padded span
      // (layers.hpp:131-132); "conv_output": "floor" opts into floor
      // semantics (= the reference on the bottom/right zero-extended input)
      if (sh < 0 || sw < 0 || (!e->conv_floor && (sh % l.stride || sw % l.stride)))
        throw ShapeMismatch("Model::validate: layer " + si +
                            " output dimensions are not positive integers for " +
                            std::to_string(s.h) + "x" + std::to_string(s.w) + " input");
      o.flat = false;
      o.c = l.c_out;
      o.h = sh / l.stride + 1;
      o.w = sw / l.stride + 1;
    } else if (l.type == L_MAXPOOL) {
      if (s.flat) throw ShapeMismatch("Model::validate: pool layer on flat input");
      o = s;
      o.h = s.h / l.window;
      o.w = s.w / l.window;
    } else if (l.type == L_AVGPOOL) {
      if (s.flat) throw ShapeMismatch("Model::validate: pool layer on flat input");
      o.d = s.c;
    } else {
      if (s.flat) throw ShapeMismatch("Model::validate: flatten on flat input");
      o.d = s.c * s.h * s.w;
      if (l.src >= 0) {  // a layer's output is stored NHWC
        o.hw = s.h * s.w;
        o.fc = s.c;
      }
    }
    if (!l.residual.empty()) {
      if (l.type != L_LINEAR && l.type != L_CONV)
        throw FormatError("model_from_descriptor: layer " + si + ": residual needs a KAN layer");
      const Named& nm = find(l.residual, si);
      if (!(nm.shape == o))
        throw ShapeMismatch("Model::validate: layer " + si + " residual '" + l.residual +
                            "' has a different shape");
      l.res_src = nm.layer;
    }
    l.out = o;
    cur = o;
    prev = idx;
    if (!l.id.empty()) {
      for (auto& kv : named)
        if (kv.first == l.id) throw FormatError("model_from_descriptor: duplicate tensor id '" + l.id + "'");
      named.push_back({l.id, {idx, o}});
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

// round a row pitch (elements) so the byte pitch is a multiple of 16 (TMA)
int64_t pitch16(int64_t n, int esz) {
  const int64_t q = 16 / esz;
  return (n + q - 1) / q * q;
}

// bytes per element of the activations a layer stores for the next one:
// u16 lattice levels on the LUT path, fp32 on the float paths
int act_esz(const kan_engine* e) { return e->cfg.mode == KAN_MODE_BSPLINE_LUT ? 2 : 4; }

// GEMM input order -> reference coefficient row (or -1 for padding).
//   conv: tap-major, then channel (im2col is channel-major, layers.hpp:140-149),
//         channels padded to whole IPS chunks per tap;
//   linear after flattening a stored NHWC tensor: pixel-major, then channel
//         (flatten is channel-major, layers.hpp:210), channels at the stored pitch;
//   otherwise the identity.
std::vector<int> input_perm(const kan_engine* e, const Layer& l, int ips, int& cps) {
  std::vector<int> perm;
  cps = 0;
  if (l.type == L_CONV && !l.im2col) {
    const int KK = l.kernel * l.kernel;
    cps = (l.c_in + ips - 1) / ips;
    const int cin_pad = cps * ips;
    perm.assign(static_cast<size_t>(KK) * cin_pad, -1);
    for (int t = 0; t < KK; ++t)
      for (int c = 0; c < l.c_in; ++c) perm[static_cast<size_t>(t) * cin_pad + c] = c * KK + t;
  } else if (l.type != L_CONV && l.in.hw > 0) {
    const int ldc = static_cast<int>(pitch16(l.in.fc, act_esz(e)));
    perm.assign(static_cast<size_t>(l.in.hw) * ldc, -1);
    for (int q = 0; q < l.in.hw; ++q)
      for (int c = 0; c < l.in.fc; ++c) perm[static_cast<size_t>(q) * ldc + c] = c * l.in.hw + q;
  } else {
    perm.resize(static_cast<size_t>(l.n_in));
    for (int i = 0; i < l.n_in; ++i) perm[static_cast<size_t>(i)] = i;
  }
  return perm;
}

void prepare_gemm_layer(kan_engine* e, const Layer& l, PreparedLayer& pl, bool bf16) {
  const kan_config& cfg = e->cfg;
  const Grid& g = e->grid;
  const int nb = g.nb();
  const int nbp = nb <= 8 ? 8 : 16;
  if (nb > 16) throw Unsupported("G + P > 16 is not supported by the tcgen05 path");
  if (g.P > 3) throw Unsupported("degree > 3 is not supported by the tcgen05 path");
  const int n_ref = l.n_in;  // reference inputs (conv: kernel^2 * c_in)
  if (l.type == L_CONV && l.kernel > 5) throw Unsupported("conv kernels larger than 5x5 are not supported");
  const int N = l.type == L_LINEAR ? l.n_out : l.c_out;
  pl.IPS = gemm_ips(bf16, nbp);
  pl.GS = gemm_gs(bf16, nbp);
  const std::vector<int> perm = input_perm(e, l, pl.IPS, pl.cps);
  const int n_in = static_cast<int>(perm.size());  // GEMM inputs
  bool holes = false;
  for (int v : perm) holes = holes || v < 0;
  pl.n_in = n_in;
  pl.N = N;
  pl.nbp = nbp;
  pl.BN = N > 256 ? 256 : std::max(16, (N + 15) / 16 * 16);
  if (const int bn = e->opt.force_bn) {  // tuning only (KAN_OPT_FORCE_BN)
    if (bn >= 16 && bn <= 256 && bn % 16 == 0 && bn < pl.BN) pl.BN = bn;
  }
  pl.n_tiles_n = (N + pl.BN - 1) / pl.BN;
  pl.silu = cfg.silu_base ? 1 : 0;
  if (pl.silu && l.base_w.size() != static_cast<size_t>(n_ref) * N)
    throw InvalidArgument("silu_base requires base weights [n_in, n_out] for every KAN layer");
  if (!bf16 && cfg.w_scheme == KAN_W_PER_TENSOR_ASYM && holes && l.type != L_CONV)
    throw Unsupported("per-tensor weights after a padded flatten are not supported");
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
        quant_joint(l.coeffs, l.base_w, static_cast<int64_t>(n_ref) * nb, n_ref, N, cfg.bits_w,
                    ratio, qw_s8, qwb, s_w);
      } else {
        quant_per_channel(l.coeffs, static_cast<int64_t>(n_ref) * nb, N, cfg.bits_w, qw_s8, s_w);
      }
      pl.b_signed = 1;
    } else {
      throw InvalidArgument("unknown weight scheme");
    }
    // int32 accumulator headroom.  The spline and SiLU parts of
    // an output share one int32 accumulator: bound |acc_j| by, per input, the
    // largest code-row sum over all lattice levels times the input's largest
    // |weight code| in column j, plus the largest SiLU code (255) times
    // |base weight code|.  Configure refuses a layer that could overflow.
    int64_t code_max = 0;
    if (e->grid.P <= 3) {
      for (int64_t a = 0; a <= e->lat.L; ++a) {
        const uint32_t v = lut_pack(e->grid, e->lat.k, e->lut, a);
        code_max = std::max<int64_t>(code_max, (v & 255u) + ((v >> 8) & 255u) + ((v >> 16) & 255u) + (v >> 24));
      }
    } else {
      code_max = static_cast<int64_t>(e->grid.P + 1) * *std::max_element(e->lut.begin(), e->lut.end());
    }
    int64_t worst = 0;
    for (int j = 0; j < N; ++j) {
      int64_t bound = 0;
      for (int ir = 0; ir < n_ref; ++ir) {
        int64_t wmax = 0;
        for (int b = 0; b < nb; ++b) {
          const size_t c = (static_cast<size_t>(ir) * nb + b) * N + j;
          wmax = std::max<int64_t>(wmax, qw_u8.empty() ? std::abs(static_cast<int64_t>(qw_s8[c])) : qw_u8[c]);
        }
        bound += code_max * wmax;
        if (!qwb.empty()) bound += 255 * std::abs(static_cast<int64_t>(qwb[static_cast<size_t>(ir) * N + j]));
      }
      worst = std::max(worst, bound);
    }
    pl.acc_bound = worst;
    if (worst > std::numeric_limits<int32_t>::max())
      throw Unsupported("KAN layer " + std::to_string(l.kan_index) + ": int32 accumulator could overflow (bound " +
                        std::to_string(worst) + " > 2^31-1); reduce n_in, lut_h or bits_w");
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
              const int ir = perm[static_cast<size_t>(i)];
              if (ir < 0) continue;
              for (int b = 0; b < nb; ++b) {
                const size_t src = (static_cast<size_t>(ir) * nb + b) * N + j;
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
              const int ir = perm[static_cast<size_t>(i)];
              if (ir < 0) continue;
              const int elem = silu_pos(bf16, nbp, gi);
              const int kb = elem * esz;
              uint8_t* dst = tile + tile_off(BN, n, kb);
              const size_t src = static_cast<size_t>(ir) * N + j;
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

  // ky-shared 3x3 stride-1 pad-1 conv kernel (kan_conv3.cuh), LUT path
  pl.conv3 = false;
  if (!bf16 && l.type == L_CONV && !l.im2col && l.kernel == 3 && l.stride == 1 && l.padding == 1 && nbp == 8 &&
      pl.b_signed && !e->opt.no_conv3) {
    const int Wo = l.out.w, Ho = l.out.h;
    if (Wo % 8 == 0 && 128 % Wo == 0 && Ho * Wo >= 128 && Ho % (128 / Wo) == 0) {
      pl.conv3 = true;
      const int cps = pl.cps;
      const int slot_raw = BN * (KSTAGE + (pl.silu ? 32 : 0));
      pl.b_slot3 = (slot_raw + 1023) / 1024 * 1024;
      std::vector<uint8_t> w3(static_cast<size_t>(pl.n_tiles_n) * 3 * 3 * cps * pl.b_slot3, 0);
      for (int nt = 0; nt < pl.n_tiles_n; ++nt)
        for (int kx = 0; kx < 3; ++kx)
          for (int cc = 0; cc < cps; ++cc)
            for (int ky = 0; ky < 3; ++ky) {
              const size_t q = (static_cast<size_t>(nt) * 3 * cps + (kx * cps + cc)) * 3 + ky;
              uint8_t* tile = w3.data() + q * pl.b_slot3;
              const int t = ky * 3 + kx;
              for (int n = 0; n < BN; ++n) {
                const int j = nt * BN + n;
                if (j >= N) continue;
                for (int ii = 0; ii < 32; ++ii) {
                  const int c = cc * 32 + ii;
                  if (c >= l.c_in) break;
                  const int ir = c * 9 + t;  // reference im2col column (layers.hpp:140-149)
                  for (int b = 0; b < nb; ++b)
                    tile[tile_off(BN, n, ii * 8 + b)] = static_cast<uint8_t>(qw_s8[(static_cast<size_t>(ir) * nb + b) * N + j]);
                  if (pl.silu) {
                    const size_t off = static_cast<size_t>(BN) * KSTAGE + (n >> 3) * 256 + (n & 7) * 32 +
                                       ((((ii >> 4) ^ ((n >> 2) & 1))) << 4) + (ii & 15);
                    tile[off] = static_cast<uint8_t>(qwb[static_cast<size_t>(ir) * N + j]);
                  }
                }
              }
            }
      pl.wt3.upload(w3);
    }
  }

  // window-shared 3x3 stride-1 pad-1 conv kernel (kan_convw.cuh): maps a
  // multiple of the tile width wide, whole 8-channel activation loads; with
  // the SiLU term, whole 32-channel groups (one SiLU block per 8 K blocks)
  pl.convw = false;
  // stride 1 (output = input size), or stride 2 onto a map a multiple of 16
  // wide (8 images per tile: every other window pixel is one core matrix)
  const int tw = std::min(16, l.out.w);  // tile width; 128 / tw images per tile
  const int cs = l.stride;
  const bool geom_ok = (cs == 1 && l.out.h == l.in.h && l.out.w == l.in.w) ||
                       (cs == 2 && tw == 16 && l.out.h == (l.in.h + 2 - 3) / 2 + 1 && l.out.w == (l.in.w + 2 - 3) / 2 + 1);
  if (!bf16 && l.type == L_CONV && !l.im2col && l.kernel == 3 && l.padding == 1 && nbp == 8 && geom_ok &&
      (!pl.silu || l.c_in % 32 == 0) && !e->opt.no_convw && l.c_in % 8 == 0 && (tw == 16 || tw == 8 || tw == 4) && l.out.w % tw == 0) {
    // N tile: 128 columns at most by default (two MMA-rate N = 128 tiles per
    // 256 channels keep the weight slots small enough for a 4-deep A ring)
    const int bn_cap = e->opt.convw_bn > 0 ? e->opt.convw_bn : 128;
    const int bnw = std::min((N + 15) / 16 * 16, bn_cap);
    const int gimg = 128 / tw;
    // output rows per tile: as many accumulators (one per row) as TMEM double-
    // buffers and the producers' window rows allow, dividing the map height
    int tr = 0;
    for (int t = 1; t <= 6; ++t)
      if (t * bnw <= 256 && l.out.h % t == 0 && ((t - 1) * cs + 3) * ((tw - 1) * cs + 3) * gimg <= convw_max_rows()) tr = t;
    if (tr > 0) {
      pl.convw = true;
      pl.bnw = bnw;
      pl.trw = tr;
      pl.ntw = (N + bnw - 1) / bnw;
      pl.b_slotw = 9 * bnw * 32;
      // ky-merged MMA issue (kan_convw.cuh): stride 1 and three N tiles' worth
      // of columns within one MMA; the taps of a kx then sit in reversed ky order
      // (pairs of taps as N = 256 MMAs for 128-column tiles were measured slower:
      // stages 2-4 +8...10 %, so the merged form stays with the <= 80-column tiles)
      pl.kymw = cs == 1 && 3 * bnw <= 256 && !e->opt.no_kym;
      const int n_kb = l.c_in / 4;
      // SiLU term: block 8 of every group of 9 holds the base weights of the
      // group's 32 channels (one byte per channel), after its 8 spline blocks
      const int n_blk = pl.silu ? n_kb + n_kb / 8 : n_kb;
      std::vector<uint8_t> ww(static_cast<size_t>(pl.ntw) * n_blk * pl.b_slotw, 0);
      for (int nt = 0; nt < pl.ntw; ++nt)
        for (int blk = 0; blk < n_blk; ++blk)
          for (int t = 0; t < 9; ++t) {
            const int tpos = pl.kymw ? (t % 3) * 3 + (2 - t / 3) : t;  // t = ky * 3 + kx
            uint8_t* tile = ww.data() + (static_cast<size_t>(nt) * n_blk + blk) * pl.b_slotw + static_cast<size_t>(tpos) * bnw * 32;
            const bool sblk = pl.silu && blk % 9 == 8;
            const int kb = pl.silu ? blk / 9 * 8 + blk % 9 : blk;  // spline K block
            for (int n = 0; n < bnw; ++n) {
              const int j = nt * bnw + n;
              if (j >= N) continue;
              for (int kbyte = 0; kbyte < 32; ++kbyte) {
                uint8_t v;
                if (sblk) {
                  const int c = blk / 9 * 32 + kbyte;
                  v = static_cast<uint8_t>(qwb[static_cast<size_t>(c * 9 + t) * N + j]);
                } else {
                  const int c = kb * 4 + kbyte / 8, b = kbyte % 8;
                  if (b >= nb) continue;
                  const int ir = c * 9 + t;  // reference im2col column (layers.hpp:140-149)
                  const size_t src = (static_cast<size_t>(ir) * nb + b) * N + j;
                  v = pl.b_signed ? static_cast<uint8_t>(qw_s8[src]) : qw_u8[src];
                }
                // SW32 K-major: 16-byte chunk c of row n at chunk c ^ (n bit 2)
                tile[n * 32 + ((((kbyte >> 4) ^ ((n >> 2) & 1))) << 4) + (kbyte & 15)] = v;
              }
            }
          }
      pl.wtw.upload(ww);
    }
  }

  // small-N layers run on CUDA cores (kan_small_layer_kernel): same integer
  // weights, laid out per (input, output) in the GEMM input order
  pl.small = !bf16 && nbp == 8 && N <= 16 && l.type == L_LINEAR && pl.b_signed &&
             static_cast<size_t>(n_in) * N * 8 <= 96 * 1024;
  if (pl.small) {
    pl.n_in8 = (n_in + 63) / 64 * 64;  // 8 threads per row x a multiple of 8 inputs each
    const int per = pl.n_in8 / 8;
    std::vector<unsigned long long> swq(static_cast<size_t>(n_in) * N, 0ull);
    std::vector<int8_t> swqb(static_cast<size_t>(N) * pl.n_in8, 0);
    for (int i = 0; i < n_in; ++i) {
      const int ir = perm[static_cast<size_t>(i)];
      if (ir < 0) continue;
      for (int j = 0; j < N; ++j) {
        unsigned long long v = 0;
        for (int b = 0; b < nb; ++b)
          v |= static_cast<unsigned long long>(static_cast<uint8_t>(qw_s8[(static_cast<size_t>(ir) * nb + b) * N + j]))
               << (8 * b);
        swq[static_cast<size_t>(i) * N + j] = v;
        // thread t = i % 8 of a row handles inputs t, t+8, ...: [j][t][e]
        if (pl.silu)
          swqb[(static_cast<size_t>(j) * 8 + i % 8) * per + i / 8] = qwb[static_cast<size_t>(ir) * N + j];
      }
    }
    swq.resize(swq.size() + 1, 0ull);  // bulk copies move whole 16-byte units
    pl.swq.upload(swq);
    std::vector<int8_t> plain((static_cast<size_t>(N) * n_in + 15) / 16 * 16, 0);
    if (pl.silu)
      for (int i = 0; i < n_in; ++i) {
        const int ir = perm[static_cast<size_t>(i)];
        if (ir < 0) continue;
        for (int j = 0; j < N; ++j) plain[static_cast<size_t>(j) * n_in + i] = qwb[static_cast<size_t>(ir) * N + j];
      }
    pl.swqb_plain.upload(plain);
    pl.swqb.upload(swqb);
  }

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
          for (int i = 0; i < n_ref; ++i) cs += qwb[static_cast<size_t>(i) * N + j];
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

// Static activation-buffer plan: a flatten is a view of its source; a stored
// tensor lives until its last consumer (next layer, input_from or residual).
void plan_buffers(kan_engine* e) {
  const int n = static_cast<int>(e->layers.size());
  std::vector<int> owner(static_cast<size_t>(n), -1), last_use(static_cast<size_t>(n), -1);
  for (int i = 0; i < n; ++i) {
    const Layer& l = e->layers[static_cast<size_t>(i)];
    owner[static_cast<size_t>(i)] = l.type == L_FLATTEN ? (l.src >= 0 ? owner[static_cast<size_t>(l.src)] : -1) : i;
  }
  for (int i = 0; i < n; ++i) {
    const Layer& l = e->layers[static_cast<size_t>(i)];
    for (int r : {l.src, l.res_src})
      if (r >= 0 && owner[static_cast<size_t>(r)] >= 0)
        last_use[static_cast<size_t>(owner[static_cast<size_t>(r)])] =
            std::max(last_use[static_cast<size_t>(owner[static_cast<size_t>(r)])], i);
  }
  e->slot_of.assign(static_cast<size_t>(n), -1);
  std::vector<int> free_slots;
  int n_slots = 0;
  for (int i = 0; i < n; ++i) {
    const Layer& l = e->layers[static_cast<size_t>(i)];
    if (l.type != L_FLATTEN && i + 1 < n) {
      int sl;
      if (!free_slots.empty()) {
        sl = free_slots.back();
        free_slots.pop_back();
      } else {
        sl = n_slots++;
      }
      e->slot_of[static_cast<size_t>(i)] = sl;
    }
    for (int j = 0; j <= i; ++j)
      if (last_use[static_cast<size_t>(j)] == i && e->slot_of[static_cast<size_t>(j)] >= 0)
        free_slots.push_back(e->slot_of[static_cast<size_t>(j)]);
  }
  e->slots.clear();
  e->slots.resize(static_cast<size_t>(n_slots));
  // storage kinds: walk backwards so a view / maxpool passes the need for
  // values on to the tensor it reads
  std::vector<bool> need(static_cast<size_t>(n), false);
  bool need_in = false;
  auto mark = [&](int t) {
    if (t >= 0)
      need[static_cast<size_t>(t)] = true;
    else if (t == -1)
      need_in = true;
  };
  for (int i = n - 1; i >= 0; --i) {
    const Layer& l = e->layers[static_cast<size_t>(i)];
    if (l.res_src != -2) mark(l.res_src);
    if (l.type == L_AVGPOOL) mark(l.src);
    if ((l.type == L_MAXPOOL || l.type == L_FLATTEN) && need[static_cast<size_t>(i)]) mark(l.src);
  }
  for (int i = 0; i < n; ++i) e->layers[static_cast<size_t>(i)].store_f32 = need[static_cast<size_t>(i)];
  e->input_f32 = need_in;
}

// ---------------------------------------------------------------------------
// Spline-table mode (EvalMode::kSplineTable, eval.hpp:17, 121-127, 137, 168):
// every KAN layer is replaced by its per-connection tables and the forward is
// table lookups + integer additions (spline_table.hpp:90-123).

static double key_to_double(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}

static void st_geometry(StLayer& sl) {
  sl.Np = sl.ft ? (sl.n_out + 3) / 4 * 16 : (sl.n_out + 15) / 16 * 16;  // bytes; 16 per lane
  const int lanes = sl.Np / 16;
  int lpr = 1;
  while (lpr < lanes && lpr < 32) lpr *= 2;
  sl.lpr = lpr;
  sl.col_tiles = (lanes + lpr - 1) / lpr;
}

// build_spline_tables (spline_table.hpp:38-95) on the device: fp64 samples in
// the reference's order, min/max fold, zero-spanning h-bit quantizer
// (RangeCalibrator + range(true) + zero_spanning, quant.hpp:79-123), quantized
// entries written straight into the gather layout.
static void st_build_layer(kan_engine* e, const Layer& l, StLayer& sl, int bits_a, int h) {
  const Grid& g = e->grid;
  const int nb = g.nb();
  const int64_t Lv = int64_t{1} << bits_a;
  std::vector<double> basis(static_cast<size_t>(Lv * nb));
  for (int64_t m = 0; m < Lv; ++m) {
    const double x = e->st_in.scale * static_cast<double>(m - e->st_in.zp);  // dequantize_value
    g.basis_at_coord(g.knot_coord(x), &basis[static_cast<size_t>(m * nb)]);
  }
  DevBuf<double> d_basis, d_coeffs;
  d_basis.upload(basis);
  d_coeffs.upload(l.coeffs);
  DevBuf<unsigned long long> mm;
  const std::vector<unsigned long long> init = {~0ull, 0ull};
  mm.upload(init);
  ck(launch_st_sample(d_basis.p, d_coeffs.p, sl.n_in, sl.n_out, nb, static_cast<int>(Lv), 0, mm.p, nullptr,
                      sl.Np, 1.0, 0.0, 0, nullptr),
     "spline table sampling");
  unsigned long long keys[2];
  ck(cudaMemcpy(keys, mm.p, sizeof(keys), cudaMemcpyDeviceToHost), "spline table range");
  if (keys[0] == ~0ull) throw InvalidArgument("calibrate_range: empty stream");
  double lo = key_to_double(keys[0]), hi = key_to_double(keys[1]);
  if (lo == hi) {  // RangeCalibrator::range(true): symmetric widening
    const double pad = std::max(std::abs(lo), 1.0) * std::numeric_limits<double>::epsilon() * 4.0;
    lo = lo - pad;
    hi = hi + pad;
  }
  lo = std::min(lo, 0.0);  // zero_spanning
  hi = std::max(hi, 0.0);
  const QParams oq = quant_params(lo, hi, h);
  sl.out_s = oq.scale;
  sl.out_z = oq.zp;
  sl.out_qhi = oq.qhi;
  sl.T.alloc(static_cast<size_t>((sl.n_in + 3) / 4 * 4) * static_cast<size_t>(Lv) * sl.Np, true);
  ck(launch_st_sample(d_basis.p, d_coeffs.p, sl.n_in, sl.n_out, nb, static_cast<int>(Lv), 1, mm.p, sl.T.p,
                      sl.Np, oq.scale, static_cast<double>(oq.zp), oq.qhi, nullptr),
     "spline table quantization");
  ck(cudaDeviceSynchronize(), "spline table build");
}

// tables supplied by the caller: reference layout [n_in][n_out][2^bits_a] ->
// gather layout [n_in][2^bits_a][Np]
static void st_import_layer(const Layer& l, StLayer& sl) {
  const int64_t Lv = int64_t{1} << l.st_bits_a;
  std::vector<uint8_t> t(static_cast<size_t>((sl.n_in + 3) / 4 * 4) * static_cast<size_t>(Lv) * sl.Np, 0);
  for (int i = 0; i < sl.n_in; ++i)
    for (int j = 0; j < sl.n_out; ++j)
      for (int64_t m = 0; m < Lv; ++m)
        t[(static_cast<size_t>(i) * Lv + m) * sl.Np + j] =
            l.st_values[(static_cast<size_t>(i) * sl.n_out + j) * Lv + m];
  sl.T.upload(t);
  sl.out_s = l.st_qd[1];
  sl.out_z = l.st_qi[2];
  sl.out_qhi = l.st_qi[3];
}

// vthr[n] = smallest integer sum v whose output s_out * v quantizes to an input
// level >= n under the consumer's quantizer (quantize_value is monotone in v);
// INT_MAX when no attainable sum reaches n.
static void st_sum_thresholds(const kan_engine* e, StLayer& sl) {
  const int64_t vmin = -static_cast<int64_t>(sl.n_in) * sl.out_z;
  const int64_t vmax = static_cast<int64_t>(sl.n_in) * (sl.out_qhi - sl.out_z);
  auto level = [&](int64_t v) { return quantize(sl.out_s * static_cast<double>(v), e->st_in); };
  std::vector<int> vt(static_cast<size_t>(e->st_in.qhi) + 1);
  vt[0] = std::numeric_limits<int>::min();
  for (int64_t n = 1; n <= e->st_in.qhi; ++n) {
    if (level(vmax) < n) {
      vt[static_cast<size_t>(n)] = std::numeric_limits<int>::max();
      continue;
    }
    int64_t lo = vmin, hi = vmax;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (level(mid) >= n)
        hi = mid;
      else
        lo = mid + 1;
    }
    vt[static_cast<size_t>(n)] = static_cast<int>(lo);
  }
  sl.vthr.upload(vt);
}

// Fake-quant mode (EvalMode::kFakeQuant, eval.hpp:106-159).  With quantized
// activations (bits_a <= 8) every input takes one of 2^bits_a values, so each
// connection's activation phi_{i,j}(level) = sum_k fq_b(basis(clamp(dequant(level))))[k]
// * fq_w(W)[i*nb+k, j] is tabulated exactly in fp64 (the reference's k order)
// and rounded once to fp32; the forward gathers and adds the fp32 entries.
// Weights: per-tensor fake quantization (maybe_fake_quant_weights, eval.hpp:70-76).
static std::vector<double> fake_quant_weights(const std::vector<double>& w, int bits) {
  if (bits == 32 || w.empty()) return w;
  double lo = w[0], hi = w[0];
  for (double v : w) {  // RangeCalibrator::observe
    lo = (v < lo) ? v : lo;
    hi = (hi < v) ? v : hi;
  }
  if (lo == hi) {
    const double pad = std::max(std::abs(lo), 1.0) * std::numeric_limits<double>::epsilon() * 4.0;
    lo -= pad;
    hi += pad;
  }
  const QParams q = quant_params(std::min(lo, 0.0), std::max(hi, 0.0), bits);
  std::vector<double> out(w.size());
  for (size_t i = 0; i < w.size(); ++i) out[i] = q.scale * static_cast<double>(quantize(w[i], q) - q.zp);
  return out;
}

void configure_fq(kan_engine* e, const kan_config& cfg) {
  const int bits_w = cfg.bits_w, bits_a = cfg.lut_k, bits_b = cfg.lut_h;
  for (int b : {bits_w, bits_a, bits_b})
    if (b != 32 && (b < 1 || b > 8)) throw InvalidArgument("compute_quant_params: bits must be in [1,8] or 32");
  if (cfg.out_kind != KAN_OUT_F32) throw InvalidArgument("int8 outputs are only produced on the LUT path");
  if (cfg.silu_base) throw InvalidArgument("fake-quant mode has no SiLU base term");
  if (e->grid.nb() > 32) throw Unsupported("fake-quant mode supports G+P <= 32");
  for (const auto& l : e->layers)
    if (l.res_src != -2 || l.type == L_AVGPOOL)
      throw Unsupported("fake-quant mode runs the reference layer set (linear, conv, maxpool, flatten)");
  if (bits_a == 32)
    throw Unsupported("fake-quant mode with passthrough activations: use bits_a <= 8 (tabulated) or mode fp32");
  const Grid& g = e->grid;
  e->st_prepass = e->opt.st_prepass;
  if (!e->a_ranges.empty() && static_cast<int>(e->a_ranges.size()) != e->n_kan)
    throw InvalidArgument("model_forward: calibrated activation policy needs a range per KAN layer");
  e->st_in = quant_params(g.lo, g.hi, bits_a);  // a_params_for, eval.hpp:55-68 (grid bounds)
  e->st_thr.upload(quant_thresholds(e->st_in));
  const int64_t Lv = int64_t{1} << bits_a;
  const int nb = g.nb();
  const QParams bq = bits_b == 32 ? QParams{} : quant_params(0.0, 1.0, bits_b);
  e->st.clear();
  e->st.resize(static_cast<size_t>(e->n_kan));
  for (const auto& l : e->layers) {
    if (l.type != L_LINEAR && l.type != L_CONV) continue;
    StLayer& sl = e->st[static_cast<size_t>(l.kan_index)];
    sl.ft = true;
    sl.n_in = l.type == L_LINEAR ? l.n_in : l.kernel * l.kernel * l.c_in;
    sl.n_out = l.type == L_LINEAR ? l.n_out : l.c_out;
    sl.bits_a = bits_a;
    sl.h = bits_b;
    // this layer's activation quantizer: grid bounds, or its calibrated range
    sl.aq = e->a_ranges.empty()
                ? e->st_in
                : quant_params(e->a_ranges[static_cast<size_t>(l.kan_index)].first,
                               e->a_ranges[static_cast<size_t>(l.kan_index)].second, bits_a);
    sl.athr.upload(quant_thresholds(sl.aq));
    sl.in_s = sl.aq.scale;
    sl.in_z = sl.aq.zp;
    sl.in_qhi = sl.aq.qhi;
    st_geometry(sl);
    if (l.coeffs.size() != static_cast<size_t>(sl.n_in) * nb * sl.n_out)
      throw InvalidArgument("coefficients of KAN layer " + std::to_string(l.kan_index) + " not set");
    // fake-quantized basis at every activation level: basis(clamp(dequant(m)))
    // (kan_linear_forward clamps, layers.hpp:111), then FakeQuantBasis at bits_b
    std::vector<double> basis(static_cast<size_t>(Lv * nb));
    for (int64_t m = 0; m < Lv; ++m) {
      const double x = g.clamp(sl.aq.scale * static_cast<double>(m - sl.aq.zp));
      double* row = &basis[static_cast<size_t>(m * nb)];
      g.basis_at_coord(g.knot_coord(x), row);
      if (bits_b != 32)
        for (int k = 0; k < nb; ++k) row[k] = bq.scale * static_cast<double>(quantize(row[k], bq) - bq.zp);
    }
    DevBuf<double> d_basis;
    d_basis.upload(basis);
    DevBuf<double> d_coeffs;
    d_coeffs.upload(fake_quant_weights(l.coeffs, bits_w));
    sl.T.alloc(static_cast<size_t>((sl.n_in + 3) / 4 * 4) * static_cast<size_t>(Lv) * sl.Np, true);
    ck(launch_st_sample(d_basis.p, d_coeffs.p, sl.n_in, sl.n_out, nb, static_cast<int>(Lv), 2, nullptr, sl.T.p,
                        sl.Np, 1.0, 0.0, 0, nullptr),
       "fake-quant table build");
    ck(cudaDeviceSynchronize(), "fake-quant table build");
  }
}

void configure_st(kan_engine* e, const kan_config& cfg) {
  const int bits_a = cfg.lut_k, h = cfg.lut_h;
  // argument checks in build_tables order (spline_table.hpp:40-43)
  if (bits_a < 1 || bits_a > 8) throw InvalidArgument("build_spline_tables: input bits must be in [1,8]");
  if (h < 2 || h > 8) throw InvalidArgument("build_spline_tables: value bits must be in [2,8]");
  if (cfg.out_kind != KAN_OUT_F32) throw InvalidArgument("int8 outputs are only produced on the LUT path");
  if (cfg.silu_base) throw InvalidArgument("spline-table mode has no SiLU base term (spline_table.hpp:14-18)");
  if (e->grid.nb() > 32) throw Unsupported("spline-table mode supports G+P <= 32");
  for (const auto& l : e->layers) {
    if (l.res_src != -2 || l.type == L_AVGPOOL)
      throw Unsupported("spline-table mode runs the reference layer set (linear, conv, maxpool, flatten)");
  }
  e->st_prepass = e->opt.st_prepass;
  e->st_in = quant_params(e->grid.lo, e->grid.hi, bits_a);  // spline_table.hpp:51
  e->st_thr.upload(quant_thresholds(e->st_in));
  e->st.clear();
  e->st.resize(static_cast<size_t>(e->n_kan));
  for (const auto& l : e->layers) {
    if (l.type != L_LINEAR && l.type != L_CONV) continue;
    StLayer& sl = e->st[static_cast<size_t>(l.kan_index)];
    sl.n_in = l.type == L_LINEAR ? l.n_in : l.kernel * l.kernel * l.c_in;  // patch_size for conv
    sl.n_out = l.type == L_LINEAR ? l.n_out : l.c_out;
    sl.bits_a = bits_a;
    sl.h = h;
    sl.in_s = e->st_in.scale;
    sl.in_z = e->st_in.zp;
    sl.in_qhi = e->st_in.qhi;
    sl.aq = e->st_in;
    st_geometry(sl);
    if (!l.st_values.empty()) {
      if (l.st_bits_a != bits_a)
        throw InvalidArgument("spline tables of KAN layer " + std::to_string(l.kan_index) +
                              " were supplied for " + std::to_string(l.st_bits_a) + " input bits");
      st_import_layer(l, sl);
    } else {
      if (l.coeffs.size() != static_cast<size_t>(sl.n_in) * e->grid.nb() * sl.n_out)
        throw InvalidArgument("coefficients of KAN layer " + std::to_string(l.kan_index) + " not set");
      st_build_layer(e, l, sl, bits_a, h);
    }
    st_sum_thresholds(e, sl);
  }
}

// Launch geometry of one spline-table launch over `rows` rows: input slices
// per row until the grid has ~1.5 CTAs per SM (measured best on C1/C2 shapes; or a slice would own fewer than
// one 4-input quad / channel), then the staged-level chunk that fits 32 KB.
static StParams st_params(const kan_engine* e, const StLayer& sl, int64_t rows = 0, int conv_c = 0) {
  StParams p{};
  p.n_in = sl.n_in;
  p.n_out = sl.n_out;
  p.Np = sl.Np;
  p.Lv = 1 << sl.bits_a;
  p.lpr = sl.lpr;
  p.col_tiles = sl.col_tiles;
  const int units = conv_c > 0 ? conv_c : (sl.n_in + 3) / 4;  // what slices split
  int S = 1;
  auto blocks = [&](int s_) { return (rows + 256 / (sl.lpr * s_) - 1) / (256 / (sl.lpr * s_)) * sl.col_tiles; };
  while (S * sl.lpr < 256 && 2 * S <= units && blocks(S) < 148 * 3 / 2) S *= 2;
  if (const int want = e->opt.st_slices) {  // tuning only (KAN_OPT_ST_SLICES)
    if (want >= 1 && (want & (want - 1)) == 0 && want * sl.lpr <= 256) S = want;
  }
  p.slices = S;
  const int RP = 256 / (sl.lpr * S);
  int ic = (32768 / RP - 8) / 8 * 8;
  ic = std::min(ic, (sl.n_in + 7) / 8 * 8);
  p.ic = std::max(ic, 8);
  p.T = sl.T.p;
  p.thr = sl.athr.p ? sl.athr.p : e->st_thr.p;
  p.inv_s = static_cast<float>(1.0 / sl.in_s);
  p.zf = static_cast<float>(sl.in_z);
  p.lvl0 = static_cast<int>(quantize(0.0, sl.aq));
  p.corr = static_cast<long long>(sl.n_in) * sl.out_z;
  p.out_s = sl.out_s;
  p.in_s = e->st_in.scale;
  p.in_zd = static_cast<double>(e->st_in.zp);
  p.in_qhi = sl.aq.qhi;
  p.vthr = sl.vthr.p;
  p.ratio_f = static_cast<float>(sl.out_s / e->st_in.scale);
  p.ft = sl.ft ? 1 : 0;
  return p;
}

struct StAct {
  const void* p = nullptr;
  bool f32 = false;  // fp32 values (the model input) or u8 levels
  int64_t ld = 0;    // dense rows: row pitch in elements (image tensors: dense NCHW)
};

// model_forward in spline-table mode (eval.hpp:200-253): u8 input levels flow
// between layers in the reference's layouts (flat rows, NCHW images); the
// model output leaves as fp32 values.
void forward_st(kan_engine* e, const float* x, int64_t M, void* out, cudaStream_t st) {
  const int nl = static_cast<int>(e->layers.size());
  StAct in;
  in.p = x;
  in.f32 = true;
  in.ld = e->input_size();
  if (e->input_shape.size() == 3) {
    bool image_use = false;
    for (const auto& l : e->layers) image_use = image_use || (l.src < 0 && l.type != L_FLATTEN);
    if (image_use) {  // conv / maxpool read u8 NCHW levels
      const int64_t n = M * e->input_size();
      e->st_xlev.alloc(static_cast<size_t>(n));
      const StLayer& s0 = e->st[0];  // the first KAN layer quantizes the model input
      ck(launch_st_levels(x, n, s0.athr.p ? s0.athr.p : e->st_thr.p, static_cast<float>(1.0 / s0.aq.scale),
                          static_cast<float>(s0.aq.zp), static_cast<int>(s0.aq.qhi), e->st_xlev.p, 0, st),
         "input levels");
      e->last_launches += 1;
      bool flat_use = false;
      for (const auto& l : e->layers) flat_use = flat_use || (l.src < 0 && l.type == L_FLATTEN);
      if (!flat_use) {
        in.p = e->st_xlev.p;
        in.f32 = false;
      } else {
        throw Unsupported("the model input cannot feed both a flatten and an image layer");
      }
    }
  }
  std::vector<StAct> acts(static_cast<size_t>(nl));
  auto slot = [&](int i, size_t bytes) -> void* {
    auto& b = e->slots[static_cast<size_t>(e->slot_of[static_cast<size_t>(i)])].main;
    b.alloc(bytes);
    return b.p;
  };
  for (int i = 0; i < nl; ++i) {
    const Layer& l = e->layers[static_cast<size_t>(i)];
    const StAct src = l.src < 0 ? in : acts[static_cast<size_t>(l.src)];
    const bool last = i + 1 == nl;
    StAct& dst = acts[static_cast<size_t>(i)];
    if (l.type == L_FLATTEN) {  // NCHW is already the reference's flatten order
      dst = src;
      dst.ld = static_cast<int64_t>(l.in.c) * l.in.h * l.in.w;
      continue;
    }
    if (l.type == L_MAXPOOL) {
      if (src.f32) throw LogicError("maxpool reads u8 levels");
      const int64_t planes = M * l.in.c;
      uint8_t* o = static_cast<uint8_t*>(slot(i, static_cast<size_t>(planes) * l.out.h * l.out.w));
      ck(launch_st_maxpool(static_cast<const uint8_t*>(src.p), planes, l.in.h, l.in.w, l.window, o, st),
         "maxpool launch");
      e->last_launches += 1;
      dst.p = o;
      dst.f32 = false;
      continue;
    }
    const StLayer& sl = e->st[static_cast<size_t>(l.kan_index)];
    const bool conv = l.type == L_CONV;
    StParams p = st_params(e, sl, conv ? M * l.out.h * l.out.w : M, conv ? l.c_in : 0);
    // a small last layer reading only this dense layer's levels runs fused:
    // one warp per row, the hidden levels never leave shared memory
    bool fused = false;
    if (!sl.ft && !conv && i + 2 == nl && sl.col_tiles == 1 && sl.n_out <= 512) {
      const Layer& nx = e->layers[static_cast<size_t>(i + 1)];
      if (nx.type == L_LINEAR && nx.src == i) {
        const StLayer& sn = e->st[static_cast<size_t>(nx.kan_index)];
        if (sn.n_out <= 16) {
          fused = true;
          p.slices = std::max(p.slices, 32 / sl.lpr);  // at least one warp per row
          p.f_on = 1;
          p.f_n_in = sn.n_in;
          p.f_n_out = sn.n_out;
          p.f_Lv = 1 << sn.bits_a;
          p.f_T = sn.T.p;
          p.f_corr = static_cast<long long>(sn.n_in) * sn.out_z;
          p.f_out_s = sn.out_s;
          p.f_out = static_cast<float*>(out);
          p.f_ld_out = sn.n_out;
        }
      }
    }
    if (conv) {
      if (src.f32) throw LogicError("conv reads u8 levels");
      p.conv = 1;
      p.rows = M * l.out.h * l.out.w;
      p.C = l.c_in;
      p.H = l.in.h;
      p.W = l.in.w;
      p.K = l.kernel;
      p.cstride = l.stride;
      p.pad = l.padding;
      p.Ho = l.out.h;
      p.Wo = l.out.w;
      p.in_kind = ST_IN_U8;
    } else {
      p.rows = M;
      p.in_kind = src.f32 ? ST_IN_F32 : ST_IN_U8;
      p.ld_x = src.ld;
    }
    p.x = src.p;
    // fp32 dense rows: quantize them once in an HBM-bound prepass (u8 levels),
    // so the gather loop reads one u32 of levels per quad instead of running
    // the threshold math and level shuffles in every lane group
    if (!conv && src.f32 && e->st_prepass && src.ld == sl.n_in) {
      const int64_t n = M * static_cast<int64_t>(sl.n_in);
      e->st_xlev.alloc(static_cast<size_t>(n));
      ck(launch_st_levels(static_cast<const float*>(src.p), n, p.thr, p.inv_s, p.zf, static_cast<int>(sl.aq.qhi),
                          e->st_xlev.p, 0, st),
         "input levels");
      e->last_launches += 1;
      p.in_kind = ST_IN_U8;
      p.x = e->st_xlev.p;
      p.ld_x = sl.n_in;
    }
    if (last) {
      p.epi = EPI_F32;
      p.out = out;
      p.ld_out = sl.n_out;
    } else {
      p.epi = EPI_LEVEL;
      // levels for the consuming KAN layer's quantizer (maxpool / flatten keep them)
      for (int j = i + 1; j < nl; ++j) {
        const Layer& lc = e->layers[static_cast<size_t>(j)];
        if (lc.type != L_LINEAR && lc.type != L_CONV) continue;
        const StLayer& sc = e->st[static_cast<size_t>(lc.kan_index)];
        p.o_thr = sc.athr.p ? sc.athr.p : e->st_thr.p;
        p.o_inv_s = static_cast<float>(1.0 / sc.aq.scale);
        p.o_zf = static_cast<float>(sc.aq.zp);
        p.o_qhi = static_cast<int>(sc.aq.qhi);
        break;
      }
      p.ld_out = conv ? 0 : (sl.n_out + 15) / 16 * 16;
      const size_t bytes = conv ? static_cast<size_t>(p.rows) * sl.n_out : static_cast<size_t>(M * p.ld_out);
      p.out = slot(i, bytes);
      dst.p = p.out;
      dst.f32 = false;
      dst.ld = conv ? 0 : p.ld_out;
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    unsigned ev_flags = cudaEventRecordDefault;
    if (e->profiling) {
      ck(cudaEventCreate(&ev0), "cudaEventCreate");
      ck(cudaEventCreate(&ev1), "cudaEventCreate");
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      ck(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
      ev_flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
      ck(cudaEventRecordWithFlags(ev0, st, ev_flags), "cudaEventRecord");
    }
    ck(launch_st_layer(p, st), "spline-table layer launch");
    e->last_launches += 1;
    if (e->profiling) {
      ck(cudaEventRecordWithFlags(ev1, st, ev_flags), "cudaEventRecord");
      e->pending.push_back({l.kan_index, ev0, ev1});
    }
    if (fused) break;  // the output layer ran inside this launch
  }
}

void configure(kan_engine* e, const kan_config* c) {
  if (!c) throw InvalidArgument("configure: null config");
  DeviceGuard dg(e->device);
  const kan_config cfg = *c;
  if (cfg.mode != KAN_MODE_FP32 && cfg.mode != KAN_MODE_BF16 && cfg.mode != KAN_MODE_BSPLINE_LUT &&
      cfg.mode != KAN_MODE_SPLINE_TABLE && cfg.mode != KAN_MODE_FAKE_QUANT)
    throw InvalidArgument("unknown evaluation mode");
  e->cfg = cfg;
  e->configured = false;
  const Layer& lastl = e->layers.back();
  if (lastl.type != L_LINEAR && lastl.type != L_CONV)
    throw Unsupported("the last layer must be a KAN layer");
  if (cfg.mode == KAN_MODE_FP32) {
    for (auto& l : e->layers)
      if (l.type == L_AVGPOOL || l.src != static_cast<int>(&l - e->layers.data()) - 1 || l.res_src != -2)
        throw Unsupported("fp32 mode runs the reference layer set (linear, conv, maxpool, flatten); "
                          "residual blocks and global pooling run on the bf16 and bspline-lut paths");
  }
  if (lastl.type == L_CONV && cfg.out_kind == KAN_OUT_I8)
    throw InvalidArgument("int8 outputs are produced by linear output layers only");
  plan_buffers(e);
  if (cfg.mode == KAN_MODE_FAKE_QUANT && cfg.lut_k == 32 && cfg.lut_h == 32) {
    // weights-only fake quantization: the fp32 Cox-de Boor path on the
    // fake-quantized coefficients (forward_linear with RecursiveBasis, eval.hpp:144-146)
    if (cfg.bits_w != 32 && (cfg.bits_w < 1 || cfg.bits_w > 8))
      throw InvalidArgument("compute_quant_params: bits must be in [1,8] or 32");
    std::vector<std::vector<double>> keep;
    for (auto& l : e->layers) {
      keep.push_back(l.coeffs);
      l.coeffs = fake_quant_weights(l.coeffs, cfg.bits_w);
    }
    kan_config c2 = cfg;
    c2.mode = KAN_MODE_FP32;
    try {
      configure(e, &c2);
    } catch (...) {
      for (size_t i = 0; i < e->layers.size(); ++i) e->layers[i].coeffs = std::move(keep[i]);
      throw;
    }
    for (size_t i = 0; i < e->layers.size(); ++i) e->layers[i].coeffs = std::move(keep[i]);
    return;
  }
  if (cfg.mode == KAN_MODE_SPLINE_TABLE || cfg.mode == KAN_MODE_FAKE_QUANT) {
    e->prep.clear();
    if (cfg.mode == KAN_MODE_SPLINE_TABLE)
      configure_st(e, cfg);
    else
      configure_fq(e, cfg);
    e->configured = true;
    return;
  }
  e->st.clear();
  const Grid& g = e->grid;
  if (cfg.mode == KAN_MODE_BSPLINE_LUT) {
    e->lut = build_lut(g.P, cfg.lut_k, cfg.lut_h);  // validates P, k, h like the reference
    if (!e->c_lut.empty() && e->c_lut_k == cfg.lut_k && e->c_lut_h == cfg.lut_h) {
      if (e->c_lut.size() != e->lut.size())
        throw FormatError("configure: the container's LUT has " + std::to_string(e->c_lut.size()) +
                          " entries, expected " + std::to_string(e->lut.size()));
      e->lut = e->c_lut;  // the caller's table (eval.hpp:40 EvalOptions::lut)
    }
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
    // then the exact level thresholds, then the SiLU codes, then (NBP = 8)
    // the per-level 8-byte code rows
    auto a16 = [](size_t n) { return (n + 15) / 16 * 16; };
    const size_t nfrac = size_t{1} << cfg.lut_k;
    std::vector<uint32_t> vals(nfrac);
    for (size_t f = 0; f < nfrac; ++f)
      vals[f] = lut_pack(g, cfg.lut_k, e->lut, static_cast<int64_t>(f));  // jj = 0
    for (int variant = 0; variant < 3; ++variant) {
      auto& ts = e->tabs[variant];
      if (variant >= 1 && g.nb() > 8) {
        ts.bytes = 0;
        continue;
      }
      const size_t rep = variant >= 1 ? 32 : 1;  // copies, interleaved by lane
      std::vector<uint8_t> blob(a16(nfrac * 4 * rep), 0);
      for (size_t f = 0; f < nfrac; ++f)
        for (size_t l = 0; l < rep; ++l) std::memcpy(&blob[(f * rep + l) * 4], &vals[f], 4);
      ts.off_thr = static_cast<int>(blob.size());
      blob.resize(a16(blob.size() + thr.size() * 4), 0);
      std::memcpy(&blob[static_cast<size_t>(ts.off_thr)], thr.data(), thr.size() * 4);
      ts.off_silu = static_cast<int>(blob.size());
      if (!codes.empty()) {
        if (variant != 1) {
          blob.insert(blob.end(), codes.begin(), codes.end());
        } else {  // 4 codes per word, word w of lane l at (w*32 + l)*4
          const size_t words = (codes.size() + 3) / 4;
          blob.resize(blob.size() + words * 32 * 4, 0);
          for (size_t a = 0; a < codes.size(); ++a)
            for (size_t l = 0; l < 32; ++l)
              blob[static_cast<size_t>(ts.off_silu) + ((a / 4) * 32 + l) * 4 + (a % 4)] = codes[a];
        }
        blob.resize(a16(blob.size()), 0);
      }
      ts.off_c64 = static_cast<int>(blob.size());
      if (variant == 0 && g.nb() <= 8) {  // NBP = 8: one 8-byte code row per level
        blob.resize(blob.size() + static_cast<size_t>(L + 1) * 8, 0);
        for (int64_t a = 0; a <= L; ++a) {
          const uint64_t v = static_cast<uint64_t>(lut_pack(g, cfg.lut_k, e->lut, a)) << (8 * (a >> cfg.lut_k));
          std::memcpy(&blob[static_cast<size_t>(ts.off_c64) + static_cast<size_t>(a) * 8], &v, 8);
        }
        blob.resize(a16(blob.size()), 0);  // cp.async.bulk sizes are multiples of 16 bytes
      }
      if (blob.size() % 16 != 0) throw LogicError("table blob must be a multiple of 16 bytes");
      ts.bytes = static_cast<int>(blob.size());
      ts.buf.upload(blob);
    }
    if (cfg.w_scheme == KAN_W_PER_TENSOR_ASYM && (cfg.bits_w < 1 || cfg.bits_w > 8))
      throw InvalidArgument("compute_quant_params: bits must be in [1,8] or 32");
  } else {
    if (cfg.mode == KAN_MODE_FP32 && cfg.out_kind != KAN_OUT_F32)
      throw InvalidArgument("int8 outputs are only produced on the LUT path");
  }
  for (auto& l : e->layers) {
    const int ncol = l.c_in * l.kernel * l.kernel;
    l.im2col = cfg.mode == KAN_MODE_BSPLINE_LUT && l.type == L_CONV && l.src == -1 && l.c_in < 16 &&
               ncol <= 64 && e->input_shape.size() == 3 && !e->opt.no_im2col;
  }
  e->prep.clear();
  e->prep.resize(static_cast<size_t>(e->n_kan));
  // tuning switches (kan_engine_set_option), read once per configure
  e->timeline = e->opt.timeline;
  e->dbg_flags = e->opt.dbg_flags;
  e->force_tab = e->opt.tables;
  e->epi_stage = e->opt.epi_stage;
  e->conv3_mc = e->opt.conv3_mc;
  e->lv_sidecar = e->opt.lv_sidecar;
  // off by default: on C3 the prepass saves layer 0 ~50 us but costs ~260 us
  // itself (measured); the path stays available and tested
  e->prepass_min = e->opt.level_prepass_min;
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
void pick_stages(bool bf16, int nbp, int BN, int x_kind, int tab_bytes, bool silu, int nacc, int& SA,
                 int& SB, int& SX, int fused_bytes = 0) {
  const size_t budget = 232448;
  SA = gemm_tmem_slots(BN, nacc);  // the A ring lives in TMEM
  for (SB = 12; SB >= 2; --SB)
    if (gemm_smem_bytes(bf16, nbp, BN, SA, SB, SB, x_kind, tab_bytes, silu, fused_bytes) <= budget) break;
  if (SB < 2) throw Unsupported("tile configuration exceeds shared memory");
  for (SX = 24; SX > SB; --SX)
    if (gemm_smem_bytes(bf16, nbp, BN, SA, SB, SX, x_kind, tab_bytes, silu, fused_bytes) <= budget) break;
  if (gemm_smem_bytes(bf16, nbp, BN, SA, SB, SX, x_kind, tab_bytes, silu, fused_bytes) > budget) SX = SB;
}

struct LayerIO {
  const void* x;
  int x_kind;
  int64_t ld_x;  // dense: row pitch; conv: channel pitch of a stored NHWC tensor
  void* out;
  int epi;
  int64_t ld_out;
  void* out2;
  // conv input geometry (per image)
  const Layer* conv = nullptr;
  int64_t n_img = 0;
  // residual add and NCHW output
  // fused output layer (split-K launches): the next, small layer and where
  // it writes; run_gemm_layer sets `fused` when it took the layer over
  PreparedLayer* fuse = nullptr;
  void* fuse_out = nullptr;
  int fuse_epi = 0;
  bool* fused = nullptr;
  uint16_t* out_lv = nullptr;  // levels sidecar to write (EPI_F32 hidden outputs)
  int res_kind = 0;
  const void* res = nullptr;
  int64_t ld_res = 0;
  int out_hw = 0;
};

// 4D tensor map over stored NHWC conv activations: dims (C, W, H, N), box
// (IPS, Wo*s, bh*s, bn) with element strides (1, s, s, 1), so one load is one
// tap's window for the tile's output pixels.  Padded taps fall outside the
// tensor (negative or past-the-end W/H coordinates; zero fill).
static CUtensorMap make_conv_xmap(const LayerIO& io, const Layer& l, int ips, int bh, int bn) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const int H = l.in.h, W = l.in.w, Cc = l.in.c, s = l.stride, Wo = l.out.w;
  const bool f32 = io.x_kind == X_F32;
  const size_t esz = f32 ? 4 : 2;
  cuuint64_t dims[4];
  cuuint64_t strides[3];
  cuuint32_t box[4];
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  {
    const uint64_t ldc = static_cast<uint64_t>(io.ld_x);
    dims[0] = static_cast<cuuint64_t>(Cc);
    dims[1] = static_cast<cuuint64_t>(W);
    dims[2] = static_cast<cuuint64_t>(H);
    dims[3] = static_cast<cuuint64_t>(io.n_img);
    strides[0] = ldc * esz;
    strides[1] = ldc * esz * W;
    strides[2] = ldc * esz * W * H;
    box[0] = static_cast<cuuint32_t>(ips);
    box[1] = static_cast<cuuint32_t>(Wo * s);
    box[2] = static_cast<cuuint32_t>(bh * s);
    box[3] = static_cast<cuuint32_t>(bn);
    estr[1] = estr[2] = static_cast<cuuint32_t>(s);
    const size_t row_bytes = static_cast<size_t>(ips) * esz;
    sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
         : row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                           : CU_TENSOR_MAP_SWIZZLE_NONE;
  }
  for (int i = 0; i < 4; ++i)
    if (box[i] > 256) throw Unsupported("conv tile exceeds the TMA box limits");
  CUresult r = get_encode_fn()(
      &m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
      const_cast<void*>(io.x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (conv) failed (" + std::to_string(r) + ")");
  return m;
}

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
  // window-shared 3x3 conv kernel: 8 images per tile, all nine taps from one
  // expanded window (kan_convw.cuh)
  if (pl.convw && io.conv && io.x_kind == X_U16 && !io.fuse &&
      (io.epi == EPI_LEVEL || io.epi == EPI_F32) && (io.ld_x & 7) == 0 &&
      ((io.ld_out & 7) == 0 || (io.epi == EPI_F32 && io.out_hw > 0)) && (!io.res_kind || (io.ld_res & 3) == 0) &&
      (io.out_hw == 0 || (!io.res_kind && !io.out_lv)) &&
      (reinterpret_cast<uintptr_t>(io.out) & 15) == 0 && (reinterpret_cast<uintptr_t>(io.res) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(io.out_lv) & 15) == 0) {
    const Layer& l = *io.conv;
    int TR = pl.trw;
    const int BNw = pl.bnw;
    if (const int t = e->opt.convw_tr; t > 0 && t < TR && l.out.h % t == 0) TR = t;  // tuning: fewer rows per tile
    const bool zp = pl.wscheme == KAN_W_PER_TENSOR_ASYM;
    const bool wsilu = pl.silu != 0;
    // one tcgen05.commit per K block (the window slot's; it also releases the
    // weight slot): automatic for N tiles >= 128, where the MMA issue stream
    // bounds the layer (measured -2...-3.4 % there, +-1 % on 64-column tiles)
    const bool lock = (e->opt.convw_lock > 0 || (e->opt.convw_lock == 0 && BNw >= 128)) && e->opt.convw_mc <= 1;
    // activation loads: CX channels (64-byte rows where the channels allow),
    // and the deepest rings that fit, trading window height for them
    const int TW = std::min(16, l.out.w), G = 128 / TW, CS = l.stride;
    const int WPX = (TW - 1) * CS + 3;  // window columns
    struct RingPick {
      int CX, SA, SB, SX, WR, TRu;
      bool ok;
    };
    auto pick_rings = [&](int tab_bytes) {
      RingPick r{};
      int CX = l.c_in % 32 == 0 ? 32 : (l.c_in % 16 == 0 ? 16 : 8);
      int SA = 4, SB = 3, SX = 2, WR = 0;
      int TRu = TR;
      auto fits = [&] { return convw_smem_bytes(BNw, WR, CX, SA, SB, SX, tab_bytes, zp, wsilu) <= 232448; };
      for (;;) {
        WR = ((TRu - 1) * CS + 3) * WPX * G;
        SA = 4, SB = 3, SX = 2;
        if (const int rings = e->opt.convw_rings) {  // tuning: SA*100 + SB*10 + SX
          SA = rings / 100;
          SB = rings / 10 % 10;
          SX = rings % 10;
        }
        while (!fits() && SB > 2) --SB;
        while (!fits() && SA > 3) --SA;
        while (!fits() && CX > 16) CX /= 2;
        while (!fits() && SA > 2) --SA;
        while (!fits() && CX > 8) CX /= 2;
        if (fits() || TRu == 1) break;
        do { --TRu; } while (TRu > 1 && l.out.h % TRu != 0);
      }
      r.CX = CX, r.SA = SA, r.SB = SB, r.SX = SX, r.WR = WR, r.TRu = TRu;
      r.ok = fits();
      return r;
    };
    // tables: the shared per-level code rows (variant 0).  Lane-private copies
    // of vals (conflict-free lookups + a 64-bit shift) were measured slower here
    // (more producer instructions and registers; stage-1 layers +7 %)
    const RingPick rp = pick_rings(e->tabs[0].bytes);
    const int tabv = 0;
    const auto& ts = e->tabs[tabv];
    const int CX = rp.CX, SA = rp.SA, SB = rp.SB, SX = rp.SX, WR = rp.WR, TRu = rp.TRu;
    if (convw_smem_bytes(BNw, WR, CX, SA, SB, SX, ts.bytes, zp, wsilu) <= 232448) {
      p.M = static_cast<int>(io.n_img);  // images
      p.N = pl.N;
      p.BN = BNw;
      p.n_tiles_n = pl.ntw;
      p.SA = SA;
      p.SB = SB;
      p.SX = SX;
      p.nacc = TRu;
      p.splits = 1;
      // weight slots shared by a cluster of image groups (multicast): the
      // weights are re-streamed from L2 per tile, 9 taps x BN x 32 B per K block
      p.mc = e->opt.convw_mc > 0 ? e->opt.convw_mc : 1;
      p.lock = lock && SB <= SA ? 1 : 0;  // one commit per K block releases the window and the weight slot
      p.kym = pl.kymw ? 1 : 0;
      // second MMA-issuing warp (even / odd accumulators): automatic with two or
      // more N tiles (ResKAN18 stages 3-4: -2...-9 % per layer; one N tile of
      // 128 columns measured +-2 % in the reference scheme, slower with SiLU)
      p.dual = p.lock && !pl.kymw && p.mc <= 1 && TRu >= 2 && convw_dual_capable(zp ? 1 : (wsilu ? 2 : 0), io.epi, G) &&
                       (e->opt.convw_dual > 0 || (e->opt.convw_dual == 0 && pl.ntw >= 2)) ? 1 : 0;
      p.tab = ts.buf.p;
      p.tab_bytes = ts.bytes;
      p.off_thr = ts.off_thr;
      p.off_silu = ts.off_silu;
      p.off_c64 = ts.off_c64;
      p.rep = tabv;
      p.wt = pl.wtw.p;
      p.ext_rows = WR;
      p.n_ss = l.c_in / 4;
      p.b_slot = pl.b_slotw;
      p.conv = 1;
      p.H = l.in.h;
      p.W = l.in.w;
      p.bh = TRu;
      p.cstride = CS;
      p.Ho = l.out.h;       // output map
      p.pimg = l.out.w;
      p.Wo = TW;     // tile width
      p.bn_img = G;  // images per tile
      p.cps = CX;    // channels per activation load
      p.lvl0 = static_cast<int>(e->lat.quantize(0.0));
      p.epi = io.epi;
      p.out = io.out;
      p.ld_out = static_cast<int>(io.ld_out);
      p.fs = pl.fs.p;
      p.corr_b = pl.corr_b.p;
      p.f_tensor = pl.f_tensor;
      p.z_w = pl.z_w;
      p.n_lo = e->grid.lo;
      p.n_hi_open = e->grid.hi_open();
      p.n_step = e->lat.step;
      p.n_inv_step = 1.0 / e->lat.step;
      p.n_L = static_cast<int>(e->lat.L);
      p.res_kind = io.res_kind;
      p.res = io.res;
      p.ld_res = static_cast<int>(io.ld_res);
      p.out_lv = io.out_lv;
      p.ld_lv = static_cast<int>(io.ld_out);
      p.out_hw = io.out_hw;
      // 4D map over the NHWC levels with the IMAGE dimension second fastest:
      // dims (C, N, W, H), box (CX channels, 8 images, 18 columns, TR + 2 rows)
      CUtensorMap xm;
      std::memset(&xm, 0, sizeof xm);
      const uint64_t ldb = static_cast<uint64_t>(io.ld_x) * 2;
      cuuint64_t dims[4] = {static_cast<cuuint64_t>(l.c_in), static_cast<cuuint64_t>(io.n_img),
                            static_cast<cuuint64_t>(l.in.w), static_cast<cuuint64_t>(l.in.h)};
      cuuint64_t strides[3] = {ldb * l.in.w * l.in.h, ldb, ldb * l.in.w};
      cuuint32_t box[4] = {static_cast<cuuint32_t>(CX), static_cast<cuuint32_t>(G), static_cast<cuuint32_t>(WPX),
                           static_cast<cuuint32_t>((TRu - 1) * CS + 3)};
      cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
      const CUtensorMapSwizzle sw = CX == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                    : CX == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
      CUresult r = get_encode_fn()(&xm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(io.x), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (convw) failed (" + std::to_string(r) + ")");
      const size_t smem = convw_smem_bytes(BNw, WR, CX, SA, SB, SX, ts.bytes, zp, wsilu);
      if (e->opt.record_plan)
        e->plan_add("convw", pl.layer_index, p.epi, p.res_kind, p.out_lv != nullptr, p.N, BNw, 1, zp ? 1 : (wsilu ? 2 : 0),
                    p.dual ? " commits=1 issuers=2" : (p.lock ? " commits=1 issuers=1" : " commits=2 issuers=1"));
      ck(launch_convw(zp ? 1 : (wsilu ? 2 : 0), xm, p, smem, st), "convw launch");  // MODE_ZP / MODE_SILU / MODE_PLAIN
      e->last_launches += 1;
      return;
    }
  }
  // ky-shared 3x3 conv kernel: full tile grids (persistent), no zero point
  // (it pays off on stored-level inputs with full channel chunks; fp32 inputs
  // and the few-channel stem stay on the general kernel, measured faster there)
  if (pl.conv3 && io.conv && io.epi != EPI_RAW && !io.fuse && io.x_kind == X_U16 && io.conv->c_in >= 32) {
    const Layer& l = *io.conv;
    const int Wo = l.out.w, bh = 128 / Wo;
    const int tiles3 = static_cast<int>((M + 127) / 128) * pl.n_tiles_n;
    if (tiles3 >= 148) {
      const int R = (bh + 2) * Wo;
      const bool silu = pl.silu != 0;
      int variant = -1, SA = 2, SB = 0, SX = 2;
      for (int v : {2, 0}) {  // lane-private vals if it leaves >= 3 tap slots
        if (e->tabs[v].bytes == 0 || (e->force_tab >= 0 && v != e->force_tab)) continue;
        for (SB = 4; SB >= 2; --SB)
          if (conv3_smem_bytes(pl.BN, R, SA, SB, SX, io.x_kind, e->tabs[v].bytes, silu) <= 232448) break;
        if (SB >= (v == 2 ? 3 : 2)) {
          variant = v;
          break;
        }
      }
      if (variant >= 0) {
        const auto& ts = e->tabs[variant];
        p.SA = SA;
        p.SB = SB;
        p.SX = SX;
        p.nacc = 2;
        p.splits = 1;
        p.mc = e->conv3_mc;
        p.tab = ts.buf.p;
        p.tab_bytes = ts.bytes;
        p.off_thr = ts.off_thr;
        p.off_silu = ts.off_silu;
        p.off_c64 = ts.off_c64;
        p.rep = variant;
        p.wt = pl.wt3.p;
        p.ext_rows = R;
        p.n_ss = 3 * pl.cps;
        p.b_slot = pl.b_slot3;
        p.conv = 1;
        p.ksz = 3;
        p.cstride = 1;
        p.pad = 1;
        p.cps = pl.cps;
        p.H = l.in.h;
        p.W = l.in.w;
        p.Ho = l.out.h;
        p.Wo = Wo;
        p.bh = bh;
        p.bn_img = 1;
        p.tpi = l.out.h / bh;
        p.pimg = 128;
        p.lvl0 = static_cast<int>(e->lat.quantize(0.0));
        p.epi = io.epi;
        p.out = io.out;
        p.ld_out = static_cast<int>(io.ld_out);
        p.fs = pl.fs.p;
        p.corr_b = pl.corr_b.p;
        p.n_lo = e->grid.lo;
        p.n_hi_open = e->grid.hi_open();
        p.n_step = e->lat.step;
        p.n_inv_step = 1.0 / e->lat.step;
        p.n_L = static_cast<int>(e->lat.L);
        p.res_kind = io.res_kind;
        p.res = io.res;
        p.ld_res = static_cast<int>(io.ld_res);
        p.out_hw = io.out_hw;
        p.out_lv = io.out_lv;
        p.ld_lv = static_cast<int>(io.ld_out);
        // the (bh+2)-row window of one (kx, chunk): box rows bh+2, one image
        const CUtensorMap xmap3 = make_conv_xmap(io, l, pl.IPS, bh + 2, 1);
        const size_t smem = conv3_smem_bytes(pl.BN, R, SA, SB, SX, io.x_kind, ts.bytes, silu);
        if (e->opt.record_plan)
          e->plan_add("conv3", pl.layer_index, p.epi, p.res_kind, p.out_lv != nullptr, p.N, p.BN, p.splits, silu ? 2 : 0);
        ck(launch_conv3(silu ? 2 : 0, xmap3, p, smem, st), "conv3 launch");
        e->last_launches += 1;
        return;
      }
    }
  }
  // table variant: the lane-private copies when they leave deep enough rings
  int SA = 2, SB = 2, SX = 2;
  int variant = 0;
  // fp32 row-major output: the epilogue stages 32x16 blocks in smem so each
  // store instruction writes whole 64-byte row segments
  // (not with a levels sidecar: the second staged pass and its warp syncs cost
  // more than the half-sector stores; ResKAN18 stem 1.55 -> 1.42 ms)
  bool stg = !bf16 && e->epi_stage && io.epi == EPI_F32 && io.out_hw == 0 && !io.res_kind && io.out_lv == nullptr;
  const int want_tab = e->force_tab >= 0 ? e->force_tab : 2;
  if (!bf16 && want_tab > 0 && e->tabs[want_tab].bytes > 0) {
    try {
      pick_stages(bf16, pl.nbp, pl.BN, io.x_kind, e->tabs[want_tab].bytes, pl.silu != 0, 1, SA, SB, SX);
      if (SB >= 3 && SX >= 4) variant = want_tab;
    } catch (const Unsupported&) {
    }
  }
  const auto& ts = e->tabs[variant];
  const int tb = bf16 ? 0 : ts.bytes;
  // the staging buffer only when it leaves the table variant and rings intact
  if (stg) {
    try {
      pick_stages(bf16, pl.nbp, pl.BN, io.x_kind, tb, pl.silu != 0, 1, SA, SB, SX, GEMM_STG_BYTES);
      stg = SB >= 3 && (variant == 0 || SX >= 4);
    } catch (const Unsupported&) {
      stg = false;
    }
  }
  const int stg_bytes = stg ? GEMM_STG_BYTES : 0;
  pick_stages(bf16, pl.nbp, pl.BN, io.x_kind, tb, pl.silu != 0, 1, SA, SB, SX, stg_bytes);
  p.stg_on = stg ? 1 : 0;
  p.tab = ts.buf.p;
  p.tab_bytes = ts.bytes;
  p.off_thr = ts.off_thr;
  p.off_silu = ts.off_silu;
  p.off_c64 = ts.off_c64;
  p.rep = variant;
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
  // fused output layer: split-K launches (each CTA reduces whole rows, then
  // runs the small layer on them) and persistent launches (the epilogue warps
  // run it on each finished 128-row tile)
  int fused_bytes = stg_bytes;
  // (persistent fusion is opt-in: the CUDA-core small layer on 8 epilogue warps
  // is latency-bound, measured slower than its own launch on C1/C2)
  if (io.fuse && (splits > 1 || e->opt.fuse_persistent) && pl.n_tiles_n == 1 && !io.conv && io.epi == EPI_LEVEL &&
      !io.res_kind && !e->opt.no_fuse) {
    const PreparedLayer& f = *io.fuse;
    const int wq_b = (f.n_in * f.N * 8 + 15) / 16 * 16;
    const int wqb_b = f.silu ? (f.N * f.n_in + 15) / 16 * 16 : 0;
    const int fb = wq_b + wqb_b + 128 * (pl.BN + 4) * 2;  // weights + hidden-level rows (padded pitch)
    int SA2 = SA, SB2 = SB, SX2 = SX;
    bool ok = f.n_in == pl.N && pl.N % 4 == 0 && f.N <= 16 && 128 / splits >= 8 && pl.wscheme == KAN_W_PER_CHANNEL_SYM;
    if (ok) {
      try {
        pick_stages(bf16, pl.nbp, pl.BN, io.x_kind, tb, pl.silu != 0, 1, SA2, SB2, SX2, fb);
      } catch (const Unsupported&) {
        ok = false;
      }
    }
    // the split-K partials are exchanged through the (then idle) rings
    if (ok && splits > 1 && red_bytes > static_cast<size_t>(SB2) * pl.BN * KSTAGE +
                              static_cast<size_t>(SX2) * 128 * pl.IPS * (io.x_kind == X_F32 ? 4 : 2))
      ok = false;
    if (ok) {
      SA = SA2;
      SB = SB2;
      SX = SX2;
      fused_bytes = fb;
      p.f_on = 1;
      p.f_N = f.N;
      p.f_silu = f.silu;
      p.f_epi = io.fuse_epi;
      p.f_ld_out = f.N;
      p.f_wq_bytes = wq_b;
      p.f_wqb_bytes = wqb_b;
      p.f_wq = f.swq.p;
      p.f_wqb = f.silu ? f.swqb_plain.p : nullptr;
      p.f_fs = f.fs.p;
      p.f_corr = f.corr_b.p;
      p.f_out = io.fuse_out;
      if (io.fused) *io.fused = true;
    }
  }
  // persistent launches double-buffer the accumulator when TMEM allows
  p.nacc = gemm_tmem_accs(pl.BN, splits);
  if (e->opt.force_nacc1) p.nacc = 1;  // tuning only: deeper A ring
  SA = gemm_tmem_slots(pl.BN, p.nacc);
  p.SA = SA;
  p.SB = SB;
  p.SX = SX;
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
  p.n_ch = pl.n_in;
  p.out_lv = io.out_lv;
  p.ld_lv = static_cast<int>(io.ld_out);
  p.res_kind = io.res_kind;
  p.res = io.res;
  p.ld_res = static_cast<int>(io.ld_res);
  p.out_hw = io.out_hw;
  CUtensorMap xmap;
  if (io.conv) {
    // M tile = bn images x bh output rows x Wo columns (rows contiguous in M)
    const Layer& l = *io.conv;
    const int Ho = l.out.h, Wo = l.out.w;
    if (Wo > 128 || 128 % Wo != 0) throw Unsupported("conv output width must divide 128");
    int bh, bn;
    if (Ho * Wo >= 128) {
      bh = 128 / Wo;
      bn = 1;
      if (Ho % bh != 0) throw Unsupported("conv output rows must tile by 128 / width");
    } else {
      if (128 % (Ho * Wo) != 0) throw Unsupported("conv output map must divide 128 pixels");
      bh = Ho;
      bn = 128 / (Ho * Wo);
    }
    p.conv = 1;
    p.ksz = l.kernel;
    p.cstride = l.stride;
    p.pad = l.padding;
    p.cps = pl.cps;
    p.H = l.in.h;
    p.W = l.in.w;
    p.Ho = Ho;
    p.Wo = Wo;
    p.bh = bh;
    p.bn_img = bn;
    p.tpi = Ho / bh;
    p.pimg = bh * Wo;
    p.lvl0 = bf16 ? 0 : static_cast<int>(e->lat.quantize(0.0));
    p.n_ch = l.c_in;
    xmap = make_conv_xmap(io, l, pl.IPS, bh, bn);
  } else {
    xmap = make_xmap(io.x, io.x_kind, M, pl.n_in, io.ld_x, pl.IPS);
  }
  const size_t smem = gemm_smem_bytes(bf16, pl.nbp, pl.BN, SA, SB, SX, io.x_kind, tb, pl.silu != 0, fused_bytes);
  // kernel variant: 0 plain, 1 per-tensor zero point (reference scheme), 2 SiLU base
  const int mode = pl.silu ? 2 : ((!bf16 && pl.wscheme == KAN_W_PER_TENSOR_ASYM) ? 1 : 0);
  if (e->opt.record_plan)
    e->plan_add(bf16 ? "gather_bf16" : "gather", pl.layer_index, p.epi, p.res_kind, p.out_lv != nullptr, p.N, p.BN,
                p.splits, mode);
  ck(launch_gather_gemm(bf16, pl.nbp, mode, xmap, p, smem, st), "gather_gemm launch");
  e->last_launches += 1;
}

void run_small_layer(kan_engine* e, PreparedLayer& pl, int64_t M, const LayerIO& io, cudaStream_t st) {
  const auto& ts = e->tabs[0];
  SmallParams p{};
  p.M = static_cast<int>(M);
  p.n_in = pl.n_in;
  p.N = pl.N;
  p.x_kind = io.x_kind;
  p.ld_x = static_cast<int>(io.ld_x);
  p.k = e->lat.k;
  p.L = static_cast<int>(e->lat.L);
  p.mode = pl.silu ? 2 : 0;
  p.x = io.x;
  p.tab = ts.buf.p;
  p.tab_bytes = ts.off_c64;  // vals, thresholds, SiLU codes (no code rows needed)
  p.off_thr = ts.off_thr;
  p.off_silu = ts.off_silu;
  p.lo_f = static_cast<float>(-e->grid.lo / e->lat.step);  // lattice_level_tie's -lo/step
  p.inv_step_f = static_cast<float>(1.0 / e->lat.step);
  p.wq = pl.swq.p;
  p.wqb = pl.swqb.p;
  p.n_in8 = pl.n_in8;
  p.epi = io.epi;
  p.out = io.out;
  p.ld_out = static_cast<int>(io.ld_out);
  p.fs = pl.fs.p;
  p.corr_b = pl.corr_b.p;
  p.n_lo = e->grid.lo;
  p.n_hi_open = e->grid.hi_open();
  p.n_step = e->lat.step;
  p.n_inv_step = 1.0 / e->lat.step;
  p.n_L = static_cast<int>(e->lat.L);
  p.out_scale = e->cfg.out_scale;
  p.inv_out_scale = 1.0 / e->cfg.out_scale;
  if (small_smem_bytes(p) > 227 * 1024) throw Unsupported("small layer exceeds shared memory");
  ck(launch_small_layer(p, st), "small layer launch");
  e->last_launches += 1;
  if (e->opt.record_plan) e->plan_add("small_layer", pl.layer_index, p.epi, 0, 0, p.N, 0, 1, p.mode);
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

// A stored activation tensor.  Dense: [M, ld] rows.  Image: NHWC with channel
// pitch ld, except the model input, which is the caller's NCHW fp32 rows.
struct Act {
  const void* p = nullptr;
  int kind = X_F32;
  bool nchw = false;
  int64_t ld = 0;
  const uint16_t* lv = nullptr;  // levels sidecar of an fp32-stored tensor (pitch ld)
};

// model_forward in fp32 mode over conv / maxpool / flatten stacks
// (convkan_forward = im2col + kan_linear_forward, layers.hpp:126-190): NCHW
// fp32 activations, explicit im2col rows through the fp32 Cox-de Boor layer
// kernel, rows reshaped back to NCHW.
void forward_fp32_nchw(kan_engine* e, const float* x, int64_t M, void* out, cudaStream_t st) {
  const int nl = static_cast<int>(e->layers.size());
  const float* cur = x;
  int64_t ld = e->input_size();  // dense rows: pitch; images: dense NCHW per sample
  for (int i = 0; i < nl; ++i) {
    const Layer& l = e->layers[static_cast<size_t>(i)];
    const bool last = i + 1 == nl;
    if (l.type == L_FLATTEN) {
      ld = static_cast<int64_t>(l.in.c) * l.in.h * l.in.w;
      continue;
    }
    auto dst = [&](size_t elems) -> float* {
      if (last) return static_cast<float*>(out);
      auto& b = e->slots[static_cast<size_t>(e->slot_of[static_cast<size_t>(i)])].main;
      b.alloc(elems * sizeof(float));
      return reinterpret_cast<float*>(b.p);
    };
    if (l.type == L_MAXPOOL) {
      const int64_t planes = M * l.in.c;
      float* o = dst(static_cast<size_t>(planes) * l.out.h * l.out.w);
      ck(launch_maxpool_f32(cur, planes, l.in.h, l.in.w, l.window, o, st), "maxpool launch");
      e->last_launches += 1;
      cur = o;
      continue;
    }
    PreparedLayer& pl = e->prep[static_cast<size_t>(l.kan_index)];
    if (l.type == L_LINEAR) {
      float* o = dst(static_cast<size_t>(M) * pl.N);
      run_fp32_layer(e, pl, M, cur, ld, o, pl.N, st);
      cur = o;
      ld = pl.N;
      continue;
    }
    // conv: patch rows, the dense layer, NCHW output
    const int hw = l.out.h * l.out.w;
    const int64_t rows = M * hw;
    e->fp_col.alloc(static_cast<size_t>(rows) * pl.n_in);
    ck(launch_im2col_f32(cur, M, l.c_in, l.in.h, l.in.w, l.kernel, l.stride, l.padding, l.out.h, l.out.w,
                         e->fp_col.p, st),
       "im2col launch");
    e->fp_rows.alloc(static_cast<size_t>(rows) * pl.N);
    run_fp32_layer(e, pl, rows, e->fp_col.p, pl.n_in, e->fp_rows.p, pl.N, st);
    float* o = dst(static_cast<size_t>(rows) * pl.N);
    ck(launch_rows_to_nchw(e->fp_rows.p, M, hw, pl.N, o, st), "reshape launch");
    e->last_launches += 2;
    cur = o;
  }
}

// model_forward (eval.hpp:200-253): run the layer graph on the caller's stream.
// KAN layers are one fused gather-GEMM launch each; pooling layers are small
// elementwise kernels; flatten is a view (the consuming linear layer's
// coefficient rows were permuted at configure time).
void forward(kan_engine* e, const float* x, int64_t M, void* out, cudaStream_t st) {
  if (!e->configured) throw LogicError("forward: engine not configured");
  if (M < 0) throw InvalidArgument("forward: negative batch");
  DeviceGuard dg(e->device);
  e->last_launches = 0;
  e->plan.clear();
  if (M == 0) return;
  if (e->cfg.mode == KAN_MODE_SPLINE_TABLE || e->cfg.mode == KAN_MODE_FAKE_QUANT) {
    forward_st(e, x, M, out, st);
    return;
  }
  const bool lut = e->cfg.mode == KAN_MODE_BSPLINE_LUT;
  const bool fp32 = e->cfg.mode == KAN_MODE_FP32;
  if (fp32) {
    bool dense = true;
    for (const auto& l : e->layers) dense = dense && l.type == L_LINEAR;
    if (!dense || e->input_shape.size() == 3) {
      forward_fp32_nchw(e, x, M, out, st);
      return;
    }
  }
  const int esz = act_esz(e);
  // the model input: dense rows need a 16-byte pitch for TMA
  Act in;
  in.p = x;
  in.kind = X_F32;
  in.nchw = e->input_shape.size() == 3;
  in.ld = e->input_size();
  if (!in.nchw && !fp32 && (in.ld * 4) % 16 != 0) {
    const int64_t D = in.ld;
    in.ld = pitch16(D, 4);
    e->xstage.alloc(static_cast<size_t>(M * in.ld));
    ck(cudaMemcpy2DAsync(e->xstage.p, in.ld * 4, x, D * 4, D * 4, M, cudaMemcpyDeviceToDevice, st),
       "stage input");
    in.p = e->xstage.p;
  }
  const int nl = static_cast<int>(e->layers.size());
  // image models: the conv / pooling layers read NHWC, so the NCHW model input
  // is transposed once (and quantized to lattice levels on the LUT path)
  if (in.nchw) {
    bool used_as_image = false;
    for (const auto& l : e->layers)
      used_as_image = used_as_image || (l.src < 0 && l.type != L_FLATTEN && !l.im2col);
    if (used_as_image) {
      for (const auto& l : e->layers)
        if (l.src < 0 && l.type == L_FLATTEN)
          throw Unsupported("the model input cannot feed both a flatten and an image layer");
      const int C = e->input_shape[0], HW = e->input_shape[1] * e->input_shape[2];
      const bool levels = lut && !e->input_f32;
      const int isz = levels ? 2 : 4;
      const int64_t ldc = pitch16(C, isz);
      e->xnhwc.alloc(static_cast<size_t>(M * HW * ldc * isz));
      ck(launch_nchw_to_nhwc(levels, x, M, C, HW, e->xnhwc.p, static_cast<int>(ldc),
                             levels ? e->d_thr.p : nullptr,
                             levels ? static_cast<float>(-e->grid.lo / e->lat.step) : 0.f,
                             levels ? static_cast<float>(1.0 / e->lat.step) : 0.f,
                             levels ? static_cast<int>(e->lat.L) : 0, st),
         "input transpose");
      e->last_launches += 1;
      if (e->opt.record_plan) e->plan_add("nchw_to_nhwc", -1, 0, 0, levels, C, 0, 0, 0);
      in.p = e->xnhwc.p;
      in.kind = levels ? X_U16 : X_F32;
      in.nchw = false;
      in.ld = ldc;
    }
  }
  std::vector<Act> acts(static_cast<size_t>(nl));
  auto slot = [&](int i, size_t bytes) -> void* {
    auto& b = e->slots[static_cast<size_t>(e->slot_of[static_cast<size_t>(i)])].main;
    b.alloc(bytes);
    return b.p;
  };
  auto slot_lv = [&](int i, size_t elems) -> uint16_t* {
    auto& b = e->slots[static_cast<size_t>(e->slot_of[static_cast<size_t>(i)])].lv;
    b.alloc(elems);
    return b.p;
  };
  for (int i = 0; i < nl; ++i) {
    const Layer& l = e->layers[static_cast<size_t>(i)];
    const Act src = l.src < 0 ? in : acts[static_cast<size_t>(l.src)];
    const bool last = i + 1 == nl;
    Act& dst = acts[static_cast<size_t>(i)];
    if (l.type == L_FLATTEN) {
      dst = src;
      dst.lv = nullptr;
      dst.ld = src.nchw ? static_cast<int64_t>(l.in.c) * l.in.h * l.in.w
                        : static_cast<int64_t>(l.in.h) * l.in.w * src.ld;
      dst.nchw = false;
      continue;
    }
    if (l.type == L_MAXPOOL || l.type == L_AVGPOOL) {
      if (src.nchw) throw Unsupported("pooling the model input is not supported");
      const int C = l.in.c;
      const int sz = src.kind == X_U16 ? 2 : 4;
      dst.kind = src.kind;
      dst.nchw = false;
      dst.ld = pitch16(C, sz);
      if (l.type == L_MAXPOOL) {
        void* o = slot(i, static_cast<size_t>(M) * l.out.h * l.out.w * dst.ld * sz);
        ck(launch_maxpool(src.kind == X_U16, src.p, M, l.in.h, l.in.w, C, static_cast<int>(src.ld),
                          l.window, o, static_cast<int>(dst.ld), st),
           "maxpool launch");
        dst.p = o;
      } else {
        if (src.kind != X_F32) throw LogicError("average pooling reads fp32 values");
        void* o = slot(i, static_cast<size_t>(M) * dst.ld * 4);
        ck(launch_avgpool(src.p, M, l.in.h * l.in.w, C, static_cast<int>(src.ld), o,
                          static_cast<int>(dst.ld), st),
           "avgpool launch");
        dst.p = o;
      }
      e->last_launches += 1;
      if (e->opt.record_plan) e->plan_add(l.type == L_MAXPOOL ? "maxpool" : "avgpool", -1, 0, 0, 0, C, 0, 0, 0);
      continue;
    }
    // ---- KAN layer ----
    PreparedLayer& pl = e->prep[static_cast<size_t>(l.kan_index)];
    const bool conv = l.type == L_CONV;
    const int64_t rows = conv ? M * l.out.h * l.out.w : M;
    LayerIO io{};
    io.x = src.p;
    io.x_kind = src.kind;
    io.ld_x = src.ld;
    if (lut && src.lv && src.kind == X_F32) {  // the producer stored levels beside the values
      io.x = src.lv;
      io.x_kind = X_U16;
    }
    // large fp32-input dense layers: levels first (HBM-bound prepass), so the
    // gather GEMM reads 2-byte levels and its producers skip the level
    // arithmetic (small layers keep the in-kernel path: their steps are
    // latency-bound)
    if (lut && !conv && src.kind == X_F32 && !src.nchw && !(pl.small) &&
        rows * static_cast<int64_t>(pl.n_in) >= e->prepass_min) {
      const int64_t ldl = pitch16(pl.n_in, 2);
      e->xlev.alloc(static_cast<size_t>(rows * ldl));
      ck(launch_rows_to_levels(static_cast<const float*>(src.p), rows, pl.n_in, static_cast<int>(src.ld), e->xlev.p,
                               static_cast<int>(ldl), e->d_thr.p, static_cast<float>(-e->grid.lo / e->lat.step),
                               static_cast<float>(1.0 / e->lat.step), static_cast<int>(e->lat.L), st),
         "level prepass");
      e->last_launches += 1;
      if (e->opt.record_plan) e->plan_add("level_prepass", l.kan_index, 0, 0, 1, pl.n_in, 0, 0, 0);
      io.x = e->xlev.p;
      io.x_kind = X_U16;
      io.ld_x = ldl;
    }
    if (conv && l.im2col) {  // explicit level im2col of the NCHW model input
      const int ncol = l.c_in * l.kernel * l.kernel;
      const int64_t ldc = pitch16(ncol, 2);
      e->xcol.alloc(static_cast<size_t>(rows * ldc));
      ck(launch_im2col_levels(x, M, l.c_in, l.in.h, l.in.w, l.kernel, l.stride, l.padding, l.out.h, l.out.w,
                              e->xcol.p, static_cast<int>(ldc), e->d_thr.p,
                              static_cast<float>(-e->grid.lo / e->lat.step), static_cast<float>(1.0 / e->lat.step),
                              static_cast<int>(e->lat.L), static_cast<int>(e->lat.quantize(0.0)), st),
         "input im2col");
      e->last_launches += 1;
      if (e->opt.record_plan) e->plan_add("im2col_levels", l.kan_index, 0, 0, 1, ncol, 0, 0, 0);
      io.x = e->xcol.p;
      io.x_kind = X_U16;
      io.ld_x = ldc;
    } else if (conv) {
      if (src.nchw) throw LogicError("conv input must be stored NHWC");
      io.conv = &l;
      io.n_img = M;
    }
    if (l.res_src != -2) {
      if (l.res_src < 0) throw Unsupported("residual from the model input is not supported");
      const Act& r = acts[static_cast<size_t>(l.res_src)];
      if (r.kind != X_F32) throw LogicError("residual tensors are stored as fp32 values");
      io.res_kind = 2;
      io.res = r.p;
      io.ld_res = r.ld;
    }
    void* o;
    if (last) {
      o = out;
      io.ld_out = pl.N;
      io.epi = (lut && e->cfg.out_kind == KAN_OUT_I8) ? EPI_I8 : EPI_F32;
      if (conv) io.out_hw = l.out.h * l.out.w;
    } else {
      const bool levels = lut && !l.store_f32;
      const int osz = levels ? 2 : 4;
      io.ld_out = pitch16(pl.N, osz);
      o = slot(i, static_cast<size_t>(rows * io.ld_out * osz));
      io.epi = levels ? EPI_LEVEL : EPI_F32;
      // fp32-stored (residual) tensors also get their levels when a KAN layer reads them
      // (at the fp32 pitch, which must also be a 16-byte pitch for u16 rows)
      if (lut && l.store_f32 && !(pl.small && !conv) && e->lv_sidecar && pitch16(pl.N, 2) == io.ld_out) {
        bool kan_consumer = false;
        for (const auto& c : e->layers)
          kan_consumer = kan_consumer || (c.src == i && (c.type == L_CONV || c.type == L_LINEAR));
        if (kan_consumer) io.out_lv = slot_lv(i, static_cast<size_t>(rows * io.ld_out));
      }
    }
    io.out = o;
    // fuse a small last layer that reads only this layer's hidden levels
    bool fused = false;
    if (lut && !conv && !last && i + 2 == nl && io.epi == EPI_LEVEL && !(pl.small && !conv)) {
      const Layer& nx = e->layers[static_cast<size_t>(i + 1)];
      PreparedLayer& pn = e->prep[static_cast<size_t>(nx.kan_index)];
      if (nx.type == L_LINEAR && nx.src == i && nx.res_src == -2 && pn.small) {
        io.fuse = &pn;
        io.fuse_out = out;
        io.fuse_epi = e->cfg.out_kind == KAN_OUT_I8 ? EPI_I8 : EPI_F32;
        io.fused = &fused;
      }
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
    if (fp32)
      run_fp32_layer(e, pl, M, static_cast<const float*>(src.p), src.ld, static_cast<float*>(o),
                     io.ld_out, st);
    else if (pl.small && !conv)
      run_small_layer(e, pl, rows, io, st);
    else
      run_gemm_layer(e, pl, rows, io, st);
    if (e->profiling) {
      ck(cudaEventRecordWithFlags(ev1, st, ev_flags), "cudaEventRecord");
      e->pending.push_back({l.kan_index, ev0, ev1});
    }
    dst.p = o;
    dst.kind = io.epi == EPI_LEVEL ? X_U16 : X_F32;
    dst.nchw = false;
    dst.ld = io.ld_out;
    dst.lv = io.out_lv;
    if (fused) break;  // the output layer ran inside this launch
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
    if (j.has("conv_output")) {
      const std::string co = j.at("conv_output").string();
      if (co != "floor" && co != "exact") throw FormatError("model_from_descriptor: conv_output must be 'exact' or 'floor'");
      e->conv_floor = co == "floor";
    }
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
      } else if (type == "global_avgpool") {
        l.type = L_AVGPOOL;
      } else {
        throw FormatError("model_from_descriptor: unknown layer type '" + type + "'");
      }
      if (jl.has("id")) l.id = jl.at("id").string();
      if (jl.has("input_from")) l.input_from = jl.at("input_from").string();
      if (jl.has("residual")) l.residual = jl.at("residual").string();
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
    l.w_bw.reset();
    l.w_master.reset();  // (the momentum restarts with new coefficients)
    l.w_vel.reset();
    l.master_ahead = false;
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

// host copy of coefficients a device-side update (kan_engine_sgd_step) moved
static void sync_master_to_host(kan_engine* e, Layer& l) {
  if (!l.master_ahead || !l.w_master) return;
  DeviceGuard dg(e->device);
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  ck(cudaMemcpy(l.coeffs.data(), l.w_master->p, l.coeffs.size() * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
  l.master_ahead = false;
}

kan_status kan_engine_configure(kan_engine* e, const kan_config* cfg) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    for (auto& l : e->layers)
      if (l.type == L_LINEAR || l.type == L_CONV) sync_master_to_host(e, l);
    configure(e, cfg);
  });
}

kan_status kan_engine_sgd_step(kan_engine* e, int layer, const float* dcoeffs_dev, double lr, double momentum,
                               void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    Layer& l = e->kan_layer(layer);
    if (!e->configured || e->cfg.mode != KAN_MODE_FP32)
      throw InvalidArgument("sgd_step: the engine must be configured in fp32 mode");
    if (!dcoeffs_dev) throw InvalidArgument("sgd_step: null gradient");
    const int nb = e->grid.nb();
    const int n_ref = l.type == L_LINEAR ? l.n_in : l.kernel * l.kernel * l.c_in;
    const int N = l.type == L_LINEAR ? l.n_out : l.c_out;
    const long long n = static_cast<long long>(n_ref) * nb * N;
    if (l.coeffs.size() != static_cast<size_t>(n)) throw InvalidArgument("sgd_step: coefficients not set");
    DeviceGuard dg(e->device);
    if (!l.w_master) {
      l.w_master = std::make_shared<DevBuf<double>>();
      l.w_master->upload(l.coeffs);
      l.w_vel = std::make_shared<DevBuf<double>>();
      l.w_vel->alloc(static_cast<size_t>(n), true);
    }
    PreparedLayer& pl = e->prep[static_cast<size_t>(l.kan_index)];
    ck(launch_sgd_step(l.w_master->p, l.w_vel->p, dcoeffs_dev, l.w_bw ? l.w_bw->p : nullptr, pl.w32.p, n, nb, pl.nbp, N,
                       pl.Npad, lr, momentum, static_cast<cudaStream_t>(stream)),
       "sgd step launch");
    l.master_ahead = true;
  });
}

kan_status kan_engine_get_coeffs(kan_engine* e, int layer, double* out, int64_t n) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    Layer& l = e->kan_layer(layer);
    if (!out || n != static_cast<int64_t>(l.coeffs.size()))
      throw ShapeMismatch("get_coeffs: expected room for " + std::to_string(l.coeffs.size()) + " coefficients");
    sync_master_to_host(e, l);
    std::copy(l.coeffs.begin(), l.coeffs.end(), out);
  });
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

kan_status kan_engine_evaluate_accuracy(kan_engine* e, const float* x_dev, const int32_t* labels_dev,
                                        int64_t batch, double* accuracy, void* stream) {
  if (!e || !accuracy) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (batch < 0) throw InvalidArgument("evaluate_accuracy: negative batch");
    *accuracy = 0.0;  // an empty dataset scores 0 (eval.hpp:281)
    if (batch == 0) return;
    if (!x_dev || !labels_dev) throw InvalidArgument("evaluate_accuracy: null buffer");
    DeviceGuard dg(e->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    e->pred_tmp.alloc(static_cast<size_t>(batch));
    const kan_status ps = kan_engine_predict(e, x_dev, batch, e->pred_tmp.p, stream);
    if (ps != KAN_OK) throw CudaError(e->err);
    const int launches = e->last_launches;
    e->count_tmp.alloc(1);
    ck(launch_count_equal(e->pred_tmp.p, labels_dev, batch, e->count_tmp.p, st), "count launch");
    unsigned long long c = 0;
    ck(cudaMemcpyAsync(&c, e->count_tmp.p, sizeof(c), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "stream sync");
    e->last_launches = launches + 1;
    *accuracy = static_cast<double>(c) / static_cast<double>(batch);
  });
}

kan_status kan_engine_layer_levels(kan_engine* e, int layer, const float* x_dev, int64_t n,
                                   uint16_t* levels_dev, void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (!e->configured || (e->cfg.mode != KAN_MODE_BSPLINE_LUT && e->cfg.mode != KAN_MODE_SPLINE_TABLE &&
                           e->cfg.mode != KAN_MODE_FAKE_QUANT))
      throw LogicError("layer_levels: engine not configured for bspline-lut");
    (void)e->kan_layer(layer);  // one grid per model (Model::grid, layers.hpp:224-230)
    DeviceGuard dg(e->device);
    e->last_launches = 0;
    if (n == 0) return;
    if (e->cfg.mode == KAN_MODE_SPLINE_TABLE || e->cfg.mode == KAN_MODE_FAKE_QUANT) {
      ck(launch_st_levels(x_dev, n, e->st_thr.p, static_cast<float>(1.0 / e->st_in.scale),
                          static_cast<float>(e->st_in.zp), static_cast<int>(e->st_in.qhi), levels_dev, 1,
                          static_cast<cudaStream_t>(stream)),
         "levels launch");
      e->last_launches = 1;
      return;
    }
    ck(launch_levels(x_dev, n, e->d_thr.p, static_cast<float>(-e->grid.lo / e->lat.step),
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
    if (!e->configured || (e->cfg.mode != KAN_MODE_BSPLINE_LUT && e->cfg.mode != KAN_MODE_SPLINE_TABLE))
      throw LogicError("layer_accumulators: engine not configured for bspline-lut");
    if (e->cfg.mode == KAN_MODE_SPLINE_TABLE) {  // any KAN layer, as dense (im2col'd) level rows
      (void)e->kan_layer(layer);
      DeviceGuard dg(e->device);
      e->last_launches = 0;
      if (batch == 0) return;
      const StLayer& sl = e->st[static_cast<size_t>(layer)];
      cudaStream_t st = static_cast<cudaStream_t>(stream);
      e->st_probe.alloc(static_cast<size_t>(batch) * sl.n_in);
      ck(launch_u16_to_u8(levels_dev, batch * sl.n_in, e->st_probe.p, st), "levels to u8");
      StParams p = st_params(e, sl, batch);
      p.rows = batch;
      p.in_kind = ST_IN_U8;
      p.x = e->st_probe.p;
      p.ld_x = sl.n_in;
      p.epi = EPI_RAW;
      p.out = acc_s_dev;
      p.ld_out = sl.n_out;
      ck(launch_st_layer(p, st), "spline-table layer launch");
      e->last_launches = 2;
      return;
    }
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
    if (pl.small)
      run_small_layer(e, pl, batch, io, static_cast<cudaStream_t>(stream));
    else
      run_gemm_layer(e, pl, batch, io, static_cast<cudaStream_t>(stream));
  });
}

kan_status kan_engine_load(const char* path, int device, kan_engine** out) {
  if (!out || !path) return KAN_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  kan_container* c = nullptr;
  kan_status st = kan_container_load(path, &c);
  if (st != KAN_OK) {
    // surface the container's message through a handle the caller can read
    auto e = std::make_unique<kan_engine>();
    e->err = kan_container_last_error(c);
    kan_container_destroy(c);
    *out = e.release();
    return st;
  }
  st = kan_engine_create(kan_container_descriptor(c), device, out);
  if (st == KAN_OK) {
    kan_engine* e = *out;
    for (int i = 0; i < kan_container_num_kan_layers(c) && st == KAN_OK; ++i) {
      std::vector<double> w(static_cast<size_t>(kan_container_coeffs(c, i, nullptr, 0)));
      kan_container_coeffs(c, i, w.data(), static_cast<int64_t>(w.size()));
      st = kan_engine_set_coeffs(e, i, w.data(), static_cast<int64_t>(w.size()), nullptr, 0);
    }
    for (int t = 0; t < kan_container_num_spline_tables(c) && st == KAN_OK; ++t) {
      int bits_a = 0, h = 0;
      double qd[2];
      int64_t qi[4];
      std::vector<uint8_t> v(static_cast<size_t>(kan_container_spline_table(c, t, nullptr, 0, nullptr, nullptr,
                                                                           nullptr, nullptr)));
      kan_container_spline_table(c, t, v.data(), static_cast<int64_t>(v.size()), &bits_a, &h, qd, qi);
      st = kan_engine_set_spline_tables(e, t, v.data(), static_cast<int64_t>(v.size()), bits_a, h, qd, qi);
    }
    int deg = 0, k = 0, h = 0;
    const int64_t nl = kan_container_lut(c, nullptr, 0, &deg, &k, &h);
    if (st == KAN_OK && nl > 0) {
      e->c_lut.resize(static_cast<size_t>(nl));
      kan_container_lut(c, e->c_lut.data(), nl, nullptr, nullptr, nullptr);
      e->c_lut_k = k;
      e->c_lut_h = h;
      if (deg != e->grid.P) {
        e->err = "load_container: LUT degree " + std::to_string(deg) + " does not match the model's degree";
        st = KAN_ERR_FORMAT;
      }
    }
  }
  kan_container_destroy(c);
  return st;
}

kan_status kan_engine_linear_backward(kan_engine* e, int layer, const float* x_dev, int64_t batch,
                                      const float* dout_dev, float* dcoeffs_dev, float* dinputs_dev, void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    Layer& l = e->kan_layer(layer);
    if (l.type != L_LINEAR) throw Unsupported("linear_backward: linear KAN layers only");
    if (batch < 0) throw InvalidArgument("linear_backward: negative batch");
    const int nb = e->grid.nb();
    if (l.coeffs.size() != static_cast<size_t>(l.n_in) * nb * l.n_out)
      throw InvalidArgument("coefficients of KAN layer " + std::to_string(layer) + " not set");
    if (nb > 16 || e->grid.P > 3) throw Unsupported("linear_backward supports G+P <= 16 and degree <= 3");
    if (batch > 0 && (!x_dev || !dout_dev || !dcoeffs_dev)) throw InvalidArgument("linear_backward: null buffer");
    DeviceGuard dg(e->device);
    if (!l.w_bw) {
      sync_master_to_host(e, l);
      l.w_bw = std::make_shared<DevBuf<float>>();
      std::vector<float> w32(l.coeffs.begin(), l.coeffs.end());
      l.w_bw->upload(w32);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (batch == 0) {  // d_coeffs of an empty batch is zero (train.hpp:95)
      ck(cudaMemsetAsync(dcoeffs_dev, 0, l.coeffs.size() * sizeof(float), st), "memset");
      return;
    }
    BwParams p{};
    p.M = batch;
    p.n_in = l.n_in;
    p.n_out = l.n_out;
    p.G = e->grid.G;
    p.P = e->grid.P;
    p.x = x_dev;
    p.ld_x = l.n_in;
    p.dy = dout_dev;
    p.w = l.w_bw->p;
    p.dcoeffs = dcoeffs_dev;
    p.dinputs = dinputs_dev;
    p.lo = static_cast<float>(e->grid.lo);
    p.hi_open = std::nextafter(static_cast<float>(e->grid.hi), static_cast<float>(e->grid.lo));
    p.inv_delta = static_cast<float>(1.0 / e->grid.delta);
    ck(launch_linear_backward(p, st), "backward launch");
  });
}

kan_status kan_engine_conv_backward(kan_engine* e, int layer, const float* x_dev, int64_t batch,
                                    const float* dout_dev, float* dcoeffs_dev, float* dinputs_dev, void* stream) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    Layer& l = e->kan_layer(layer);
    if (l.type != L_CONV) throw Unsupported("conv_backward: conv KAN layers only");
    if (batch < 0) throw InvalidArgument("conv_backward: negative batch");
    const int nb = e->grid.nb();
    const int n_in = l.kernel * l.kernel * l.c_in;
    if (l.coeffs.size() != static_cast<size_t>(n_in) * nb * l.c_out)
      throw InvalidArgument("coefficients of KAN layer " + std::to_string(layer) + " not set");
    if (nb > 16 || e->grid.P > 3) throw Unsupported("conv_backward supports G+P <= 16 and degree <= 3");
    if (batch > 0 && (!x_dev || !dout_dev || !dcoeffs_dev)) throw InvalidArgument("conv_backward: null buffer");
    DeviceGuard dg(e->device);
    if (!l.w_bw) {
      sync_master_to_host(e, l);
      l.w_bw = std::make_shared<DevBuf<float>>();
      std::vector<float> w32(l.coeffs.begin(), l.coeffs.end());
      l.w_bw->upload(w32);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (batch == 0) {
      ck(cudaMemsetAsync(dcoeffs_dev, 0, l.coeffs.size() * sizeof(float), st), "memset");
      return;
    }
    // the reference's conv backward: im2col patches of the input, the linear
    // backward on the patch rows, col2im_add of the patch gradients
    // (train.hpp:367-399)
    const int hw = l.out.h * l.out.w;
    const int64_t rows = batch * hw;
    e->fp_col.alloc(static_cast<size_t>(rows) * n_in);
    ck(launch_im2col_f32(x_dev, batch, l.c_in, l.in.h, l.in.w, l.kernel, l.stride, l.padding, l.out.h, l.out.w,
                         e->fp_col.p, st),
       "im2col launch");
    e->bw_drows.alloc(static_cast<size_t>(rows) * l.c_out);
    ck(launch_nchw_to_rows(dout_dev, batch, hw, l.c_out, e->bw_drows.p, st), "gradient rows");
    if (dinputs_dev) e->bw_dpatch.alloc(static_cast<size_t>(rows) * n_in);
    BwParams p{};
    p.M = rows;
    p.n_in = n_in;
    p.n_out = l.c_out;
    p.G = e->grid.G;
    p.P = e->grid.P;
    p.x = e->fp_col.p;
    p.ld_x = n_in;
    p.dy = e->bw_drows.p;
    p.w = l.w_bw->p;
    p.dcoeffs = dcoeffs_dev;
    p.dinputs = dinputs_dev ? e->bw_dpatch.p : nullptr;
    p.lo = static_cast<float>(e->grid.lo);
    p.hi_open = std::nextafter(static_cast<float>(e->grid.hi), static_cast<float>(e->grid.lo));
    p.inv_delta = static_cast<float>(1.0 / e->grid.delta);
    ck(launch_linear_backward(p, st), "backward launch");
    if (dinputs_dev)
      ck(launch_col2im(e->bw_dpatch.p, batch, l.c_in, l.in.h, l.in.w, l.kernel, l.stride, l.padding, l.out.h,
                       l.out.w, dinputs_dev, st),
         "col2im launch");
  });
}

kan_status kan_maxpool2_f32(const float* in_dev, int64_t planes, int H, int W, int window, float* out_dev,
                            void* stream) {
  if (planes < 0 || window < 1 || H < window || W < window) return KAN_ERR_INVALID_ARGUMENT;
  return launch_maxpool_f32(in_dev, planes, H, W, window, out_dev, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? KAN_OK
             : KAN_ERR_CUDA;
}

kan_status kan_maxpool2_backward_f32(const float* in_dev, int64_t planes, int H, int W, int window,
                                     const float* dout_dev, float* din_dev, void* stream) {
  if (planes < 0 || window < 1 || H < window || W < window) return KAN_ERR_INVALID_ARGUMENT;
  return launch_maxpool_bw(in_dev, planes, H, W, window, dout_dev, din_dev, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? KAN_OK
             : KAN_ERR_CUDA;
}

kan_status kan_softmax_cross_entropy(const float* logits_dev, const int32_t* labels_dev, int64_t batch, int n,
                                     float* loss_rows_dev, float* dlogits_dev, void* stream) {
  if (batch < 0 || n < 1) return KAN_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!logits_dev || !labels_dev || !loss_rows_dev || !dlogits_dev)) return KAN_ERR_INVALID_ARGUMENT;
  const cudaError_t e = launch_softmax_ce(logits_dev, labels_dev, batch, n, loss_rows_dev, dlogits_dev,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KAN_OK : KAN_ERR_CUDA;
}

kan_status kan_engine_set_activation_ranges(kan_engine* e, const double* ranges, int n) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    if (n == 0) {
      e->a_ranges.clear();
    } else {
      if (n != e->n_kan || !ranges)
        throw InvalidArgument("model_forward: calibrated activation policy needs a range per KAN layer");
      e->a_ranges.clear();
      for (int i = 0; i < n; ++i) e->a_ranges.emplace_back(ranges[2 * i], ranges[2 * i + 1]);
    }
    e->configured = false;
  });
}

kan_status kan_engine_set_spline_tables(kan_engine* e, int layer, const uint8_t* values, int64_t n,
                                        int bits_a, int h, const double* qp_d, const int64_t* qp_i) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    Layer& l = e->kan_layer(layer);
    if (n == 0) {
      l.st_values.clear();
      l.st_bits_a = 0;
      return;
    }
    if (bits_a < 1 || bits_a > 8) throw InvalidArgument("build_spline_tables: input bits must be in [1,8]");
    if (h < 2 || h > 8) throw InvalidArgument("build_spline_tables: value bits must be in [2,8]");
    if (!values || !qp_d || !qp_i) throw InvalidArgument("set_spline_tables: null buffer");
    const int64_t n_in = l.type == L_LINEAR ? l.n_in : static_cast<int64_t>(l.kernel) * l.kernel * l.c_in;
    const int64_t n_out = l.type == L_LINEAR ? l.n_out : l.c_out;
    if (n != (n_in * n_out) << bits_a)
      throw ShapeMismatch("set_spline_tables: expected " + std::to_string((n_in * n_out) << bits_a) +
                          " entries, got " + std::to_string(n));
    if (!(qp_d[1] > 0.0) || qp_i[3] != (int64_t{1} << h) - 1)
      throw InvalidArgument("set_spline_tables: output quantizer does not match the value bits");
    l.st_values.assign(values, values + n);
    l.st_bits_a = bits_a;
    l.st_h = h;
    l.st_qd[0] = qp_d[0];
    l.st_qd[1] = qp_d[1];
    for (int t = 0; t < 4; ++t) l.st_qi[t] = qp_i[t];
    e->configured = false;
  });
}

int64_t kan_engine_spline_table(kan_engine* e, int layer, uint8_t* out, int64_t cap, double* qp_d,
                                int64_t* qp_i) {
  if (!e) return -KAN_ERR_INVALID_ARGUMENT;
  int64_t count = 0;
  const kan_status s = guarded(e, [&] {
    if (!e->configured || e->cfg.mode != KAN_MODE_SPLINE_TABLE)
      throw LogicError("spline_table: engine not configured for spline-table mode");
    (void)e->kan_layer(layer);
    const StLayer& sl = e->st[static_cast<size_t>(layer)];
    const int64_t Lv = int64_t{1} << sl.bits_a;
    count = static_cast<int64_t>(sl.n_in) * sl.n_out * Lv;
    if (qp_d) {
      qp_d[0] = sl.in_s;
      qp_d[1] = sl.out_s;
    }
    if (qp_i) {
      qp_i[0] = sl.in_z;
      qp_i[1] = sl.in_qhi;
      qp_i[2] = sl.out_z;
      qp_i[3] = sl.out_qhi;
    }
    if (!out || cap < count) return;
    DeviceGuard dg(e->device);
    std::vector<uint8_t> t(static_cast<size_t>(sl.n_in) * Lv * sl.Np);
    ck(cudaMemcpy(t.data(), sl.T.p, t.size(), cudaMemcpyDeviceToHost), "spline table D2H");
    for (int i = 0; i < sl.n_in; ++i)
      for (int j = 0; j < sl.n_out; ++j)
        for (int64_t m = 0; m < Lv; ++m)
          out[(static_cast<int64_t>(i) * sl.n_out + j) * Lv + m] = t[(static_cast<size_t>(i) * Lv + m) * sl.Np + j];
  });
  return s == KAN_OK ? count : -static_cast<int64_t>(s);
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

kan_status kan_engine_set_option(kan_engine* e, int option, int64_t value) {
  if (!e) return KAN_ERR_INVALID_ARGUMENT;
  return guarded(e, [&] {
    auto& o = e->opt;
    const int v = static_cast<int>(value);
    switch (option) {
      case KAN_OPT_NO_CONV3: o.no_conv3 = value != 0; break;
      case KAN_OPT_NO_CONVW: o.no_convw = value != 0; break;
      case KAN_OPT_CONVW_RINGS: o.convw_rings = v; break;
      case KAN_OPT_CONVW_TR: o.convw_tr = v; break;
      case KAN_OPT_CONVW_BN:
        if (v != 0 && (v < 16 || v > 256 || v % 16)) throw InvalidArgument("KAN_OPT_CONVW_BN: 0 or a multiple of 16 in 16..256");
        o.convw_bn = v;
        break;
      case KAN_OPT_NO_FUSE: o.no_fuse = value != 0; break;
      case KAN_OPT_CONVW_NO_KYM: o.no_kym = value != 0; break;
      case KAN_OPT_FUSE_PERSISTENT: o.fuse_persistent = value != 0; break;
      case KAN_OPT_CONVW_LOCK:
        if (v < -1 || v > 1) throw InvalidArgument("KAN_OPT_CONVW_LOCK: -1, 0 or 1");
        o.convw_lock = v;
        break;
      case KAN_OPT_CONVW_DUAL:
        if (v < -1 || v > 1) throw InvalidArgument("KAN_OPT_CONVW_DUAL: -1, 0 or 1");
        o.convw_dual = v;
        break;
      case KAN_OPT_CONVW_MC:
        if (v < 0 || v > 4 || v == 3) throw InvalidArgument("KAN_OPT_CONVW_MC: 0 (auto), 1, 2 or 4");
        o.convw_mc = v;
        break;
      case KAN_OPT_NO_IM2COL: o.no_im2col = value != 0; break;
      case KAN_OPT_FORCE_BN: o.force_bn = v; break;
      case KAN_OPT_TABLES:
        if (v < -1 || v > 2) throw InvalidArgument("KAN_OPT_TABLES: -1, 0, 1 or 2");
        o.tables = v;
        break;
      case KAN_OPT_EPI_STAGE: o.epi_stage = value != 0; break;
      case KAN_OPT_CONV3_MC:
        if (v < 1 || v > 2) throw InvalidArgument("KAN_OPT_CONV3_MC: 1 or 2");
        o.conv3_mc = v;
        break;
      case KAN_OPT_LV_SIDECAR: o.lv_sidecar = value != 0; break;
      case KAN_OPT_LEVEL_PREPASS_MIN:
        o.level_prepass_min = value >= 0 ? value : std::numeric_limits<int64_t>::max();
        break;
      case KAN_OPT_ST_PREPASS: o.st_prepass = value != 0; break;
      case KAN_OPT_ST_SLICES: o.st_slices = v; break;
      case KAN_OPT_TIMELINE: o.timeline = value != 0; break;
      case KAN_OPT_FORCE_NACC1: o.force_nacc1 = value != 0; break;
      case KAN_OPT_RECORD_PLAN: o.record_plan = value != 0; break;
      case KAN_OPT_DBG_FLAGS: o.dbg_flags = v; break;
      default: throw InvalidArgument("unknown engine option " + std::to_string(option));
    }
  });
}

const char* kan_engine_last_plan(const kan_engine* e) { return e ? e->plan.c_str() : ""; }

void kan_shard_rows(int64_t batch, int g, int n, int64_t* start, int64_t* stop) {
  const int64_t per = n > 0 ? (batch + n - 1) / n : 0;
  const int64_t s = std::min(batch, static_cast<int64_t>(g) * per);
  if (start) *start = s;
  if (stop) *stop = std::min(batch, s + per);
}

namespace {
// bytes of one output row of a configured engine
size_t out_row_bytes(kan_engine* e) {
  const bool i8 = e->cfg.mode == KAN_MODE_BSPLINE_LUT && e->cfg.out_kind == KAN_OUT_I8;
  return static_cast<size_t>(e->output_count()) * (i8 ? 1 : 4);
}

void check_shard_group(kan_engine* const* engines, int n, int64_t batch) {
  if (!engines || n < 1) throw InvalidArgument("forward_sharded: no engines");
  if (batch < 0) throw InvalidArgument("forward_sharded: negative batch");
  kan_engine* e0 = engines[0];
  for (int g = 0; g < n; ++g) {
    kan_engine* e = engines[g];
    if (!e) throw InvalidArgument("forward_sharded: null engine");
    if (!e->configured) throw LogicError("forward_sharded: engine not configured");
    if (e->input_size() != e0->input_size() || out_row_bytes(e) != out_row_bytes(e0) ||
        e->cfg.mode != e0->cfg.mode)
      throw ShapeMismatch("forward_sharded: engines must run the same model and configuration");
    for (int h = 0; h < g; ++h)
      if (engines[h] == e) throw InvalidArgument("forward_sharded: an engine appears twice (one handle per shard)");
  }
}

// peer access from device `from` to device `to` (idempotent; absent P2P the
// copy engine still moves the bytes through cudaMemcpyPeerAsync)
void enable_peer(int from, int to) {
  if (from == to) return;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, from, to) != cudaSuccess || !can) return;
  DeviceGuard dg(from);
  const cudaError_t r = cudaDeviceEnablePeerAccess(to, 0);
  if (r != cudaSuccess) cudaGetLastError();  // already enabled: clear the sticky-free error
}
}  // namespace

kan_status kan_engine_forward_sharded(kan_engine* const* engines, int n_engines, const float* const* x_shards,
                                      int64_t batch, void* out_dev0, void* const* streams) {
  if (!engines || n_engines < 1 || !engines[0]) return KAN_ERR_INVALID_ARGUMENT;
  kan_engine* e0 = engines[0];
  return guarded(e0, [&] {
    check_shard_group(engines, n_engines, batch);
    if (batch > 0 && !out_dev0) throw InvalidArgument("forward_sharded: null output");
    const size_t ob = out_row_bytes(e0);
    const int dev0 = e0->device;
    cudaStream_t st0 = streams ? static_cast<cudaStream_t>(streams[0]) : nullptr;
    for (int g = 0; g < n_engines; ++g) {
      kan_engine* e = engines[g];
      int64_t r0 = 0, r1 = 0;
      kan_shard_rows(batch, g, n_engines, &r0, &r1);
      const int64_t rows = r1 - r0;
      if (rows > 0 && (!x_shards || !x_shards[g])) throw InvalidArgument("forward_sharded: null input shard");
      DeviceGuard dg(e->device);
      cudaStream_t st = streams ? static_cast<cudaStream_t>(streams[g]) : nullptr;
      uint8_t* dst = static_cast<uint8_t*>(out_dev0) + static_cast<size_t>(r0) * ob;
      const bool in_place = e->device == dev0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
      void* o = dst;
      if (!in_place && rows > 0) {
        e->shard_out.alloc(static_cast<size_t>(rows) * ob);
        o = e->shard_out.p;
      }
      forward(e, rows > 0 ? x_shards[g] : nullptr, rows, o, st);
      if (!in_place && rows > 0) {
        if (e->device == dev0)
          ck(cudaMemcpyAsync(dst, o, static_cast<size_t>(rows) * ob, cudaMemcpyDeviceToDevice, st), "shard copy");
        else {
          enable_peer(e->device, dev0);
          ck(cudaMemcpyPeerAsync(dst, dev0, o, e->device, static_cast<size_t>(rows) * ob, st), "peer copy");
        }
      }
      if (g > 0 || st != st0) {
        ck(cudaEventRecord(e->done_event(), st), "event record");
        DeviceGuard d0(dev0);
        ck(cudaStreamWaitEvent(st0, e->shard_done, 0), "stream wait");
      }
    }
  });
}

kan_status kan_engine_forward_sharded_host(kan_engine* const* engines, int n_engines, const float* x_host,
                                           int64_t batch, void* out_host) {
  if (!engines || n_engines < 1 || !engines[0]) return KAN_ERR_INVALID_ARGUMENT;
  kan_engine* e0 = engines[0];
  return guarded(e0, [&] {
    check_shard_group(engines, n_engines, batch);
    if (batch > 0 && (!x_host || !out_host)) throw InvalidArgument("forward_sharded_host: null buffer");
    const size_t ob = out_row_bytes(e0);
    const int64_t D = e0->input_size();
    // enqueue every shard (H2D, forward, D2H on the engine's own stream), then wait
    for (int g = 0; g < n_engines; ++g) {
      kan_engine* e = engines[g];
      int64_t r0 = 0, r1 = 0;
      kan_shard_rows(batch, g, n_engines, &r0, &r1);
      const int64_t rows = r1 - r0;
      if (rows <= 0) continue;
      DeviceGuard dg(e->device);
      cudaStream_t st = e->stream_own();
      e->io_in.alloc(static_cast<size_t>(rows * D) * 4);
      e->io_out.alloc(static_cast<size_t>(rows) * ob);
      ck(cudaMemcpyAsync(e->io_in.p, x_host + r0 * D, static_cast<size_t>(rows * D) * 4, cudaMemcpyHostToDevice, st),
         "H2D");
      forward(e, reinterpret_cast<const float*>(e->io_in.p), rows, e->io_out.p, st);
      ck(cudaMemcpyAsync(static_cast<uint8_t*>(out_host) + static_cast<size_t>(r0) * ob, e->io_out.p,
                         static_cast<size_t>(rows) * ob, cudaMemcpyDeviceToHost, st),
         "D2H");
    }
    for (int g = 0; g < n_engines; ++g) {
      kan_engine* e = engines[g];
      if (!e->own_stream) continue;
      DeviceGuard dg(e->device);
      ck(cudaStreamSynchronize(e->own_stream), "stream sync");
    }
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

int64_t kan_spline_thresholds(double lo, double hi, int bits_a, float* out, int64_t cap) {
  try {
    if (bits_a < 1 || bits_a > 8) return -KAN_ERR_INVALID_ARGUMENT;
    const auto thr = quant_thresholds(quant_params(lo, hi, bits_a));
    const int64_t n = static_cast<int64_t>(thr.size());
    if (out && cap >= n) std::memcpy(out, thr.data(), static_cast<size_t>(n) * sizeof(float));
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
