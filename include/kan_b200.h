/*
 * kan_b200.h -- C ABI of the B200-native KAN inference engine.
 *
 * Drop-in boundary for the reference's KAN-layer forward path
 * (reference = arxiv/paper_2603_17230 "KANtize", proj/include/kantize/).
 * Plain pointers and sizes only: no torch, no C++ types, no exceptions cross
 * this boundary.  Errors are status codes plus a per-engine message.
 *
 * Reference interface each entry point replaces:
 *   kan_engine_create           model_from_descriptor(json)       io.hpp:357-386
 *                               (+ Model::validate)                layers.hpp:252-307
 *   kan_engine_set_coeffs       KanLinearLayer/ConvKanLayer::coeffs layers.hpp:18-64
 *                               (row layout i*(G+P)+k, layers.hpp:15-17, 36-38)
 *   kan_engine_configure        EvalOptions{mode, qcfg.bits_w, lut} eval.hpp:37-45,
 *                               build_bspline_lut(P, k, h)          lut.hpp:103-131,
 *                               PreparedModel::make (W quant once)  eval.hpp:83-132
 *   kan_engine_forward          model_forward(model, inputs, opts)  eval.hpp:200-253
 *   kan_engine_forward_host     same, host buffers (H2D + D2H inside)
 *   kan_engine_predict          predict(model, inputs, opts)        eval.hpp:255-276
 *   kan_engine_evaluate_accuracy  evaluate_accuracy(model, ds, opts) eval.hpp:279-287
 *   kan_engine_layer_levels     ActivationLattice::quantize(clamp)  lut.hpp:44-47
 *   kan_engine_layer_accumulators  the int32 form of the contraction behind
 *                               tabulated_kan_forward               lut.hpp:217-231
 *   kan_lut_build               build_bspline_lut                   lut.hpp:103-131
 *   kan_engine_set_spline_tables  EvalOptions::tables (SplineTableSet) eval.hpp:41,
 *                               spline_table.hpp:19-34
 *   kan_engine_spline_table     build_spline_tables (probe)         spline_table.hpp:38-95
 *   kan_container_load / _save  load_container / save_container     io.hpp:99-350
 *   kan_engine_load             load_model / load_container + engine io.hpp:217-352
 *   kan_engine_linear_backward  kan_linear_backward                 train.hpp:84-136
 *   kan_softmax_cross_entropy   softmax_cross_entropy               train.hpp:139-160
 *
 * Error mapping (reference exception -> status):
 *   std::invalid_argument (bits, LUT params, mode)  -> KAN_ERR_INVALID_ARGUMENT
 *     quant.hpp:35-38, lut.hpp:104-106, eval.hpp:24
 *   std::invalid_argument (shape checks)            -> KAN_ERR_SHAPE_MISMATCH
 *     layers.hpp:102-105, 131-132, 252-307, eval.hpp:213-214
 *   std::out_of_range (lattice level)               -> KAN_ERR_OUT_OF_RANGE  lut.hpp:142-143
 *   io_error / format_error / checksum_error        -> KAN_ERR_IO / _FORMAT / _CHECKSUM
 *     io.hpp:21-29
 *   std::logic_error                                -> KAN_ERR_LOGIC  eval.hpp:160
 *
 * Threading: a handle is used by one host thread at a time (the reference's
 * forward is reentrant over const inputs; here one handle
 * per thread or external synchronization).  One handle binds one device.
 */
#ifndef KAN_B200_H
#define KAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kan_engine kan_engine;

typedef enum {
  KAN_OK = 0,
  KAN_ERR_INVALID_ARGUMENT = 1,
  KAN_ERR_SHAPE_MISMATCH = 2,
  KAN_ERR_OUT_OF_RANGE = 3,
  KAN_ERR_CUDA = 4,
  KAN_ERR_NCCL = 5,
  KAN_ERR_IO = 6,
  KAN_ERR_FORMAT = 7,
  KAN_ERR_CHECKSUM = 8,
  KAN_ERR_UNSUPPORTED = 9,
  KAN_ERR_LOGIC = 10
} kan_status;

/* Forward datapaths (EvalMode, eval.hpp:17; BF16 is new, FP32 = kFp32,
 * BSPLINE_LUT = kBsplineLut, SPLINE_TABLE = kSplineTable). */
typedef enum {
  KAN_MODE_FP32 = 0,         /* fp32 Cox-de Boor basis + fp32 FFMA contraction */
  KAN_MODE_BF16 = 1,         /* fp32 basis -> bf16, tcgen05 kind::f16, fp32 accumulate */
  KAN_MODE_BSPLINE_LUT = 2,  /* lattice + quantized LUT, tcgen05 kind::i8, int32 accumulate */
  KAN_MODE_SPLINE_TABLE = 3, /* per-connection spline tables, gather + integer add
                                (spline_table.hpp:19-123); lut_k = input bits bits_a,
                                lut_h = value bits h */
  KAN_MODE_FAKE_QUANT = 4    /* EvalMode::kFakeQuant (eval.hpp:106-159): bits_w per-tensor
                                weights, lut_k = bits_a (grid-bound activation quantizer),
                                lut_h = bits_b (basis over [0,1]); 32 = passthrough.
                                bits_a <= 8: exact fp64 per-connection fp32 tables, gather
                                + fp32 add; bits_a = bits_b = 32: the fp32 Cox-de Boor path */
} kan_mode;

/* Weight quantization on the LUT path. */
typedef enum {
  KAN_W_PER_TENSOR_ASYM = 0,  /* the reference's scheme (eval.hpp:70-76): u8 + zero point */
  KAN_W_PER_CHANNEL_SYM = 1   /* per output channel, symmetric, s8/s4 (engine extension) */
} kan_wscheme;

typedef enum {
  KAN_OUT_F32 = 0, /* fp32 logits */
  KAN_OUT_I8 = 1   /* int8 logits: clamp(llround(y / out_scale), -127, 127) */
} kan_out_kind;

typedef struct {
  int mode;         /* kan_mode */
  int lut_k;        /* LUT address bits per knot interval, 1..8 (lut.hpp:22);
                       spline-table mode: input address bits bits_a, 1..8 */
  int lut_h;        /* LUT value bits, 2..8 (lut.hpp:75); spline-table mode: h */
  int bits_w;       /* weight bits: 1..8 per-tensor, 2..8 per-channel (8 and 4 tested) */
  int w_scheme;     /* kan_wscheme */
  int silu_base;    /* 1: add SiLU(x) . w_base (needs kan_engine_set_coeffs base weights) */
  int out_kind;     /* kan_out_kind */
  double out_scale; /* int8 logits scale (out_kind == KAN_OUT_I8) */
  int split_k;      /* 0 = automatic; >= 1 forces the number of K splits per layer */
} kan_config;

/* Build an engine from the reference's descriptor JSON schema
 * ({name, grid{intervals,degree}, input[], [domain[lo,hi]], layers[...]},
 * io.hpp:357-386).  Coefficients start at zero, as model_from_descriptor does. */
kan_status kan_engine_create(const char* descriptor_json, int device, kan_engine** out);
void kan_engine_destroy(kan_engine* e);
const char* kan_engine_last_error(const kan_engine* e);

/* Number of KAN (linear/conv) layers; input feature count (prod of input[]);
 * output count (Model::output_count, layers.hpp:236-242). */
int kan_engine_num_kan_layers(const kan_engine* e);
int64_t kan_engine_input_size(const kan_engine* e);
int kan_engine_output_count(const kan_engine* e);
/* shape of KAN layer i: n_in (patch size for conv) and n_out */
kan_status kan_engine_layer_shape(const kan_engine* e, int layer, int* n_in, int* n_out);

/* Host fp64 coefficients of KAN layer `layer` in the reference row layout
 * [n_in*(G+P), n_out] (layers.hpp:15-17); base_w: [n_in, n_out] or NULL. */
kan_status kan_engine_set_coeffs(kan_engine* e, int layer, const double* coeffs, int64_t n,
                                 const double* base_w, int64_t n_base);

/* Quantize / convert weights once, build tables, upload (PreparedModel::make). */
kan_status kan_engine_configure(kan_engine* e, const kan_config* cfg);

/* model_forward on device buffers: x [batch, input_size] fp32 row-major (image
 * models: CHW per row, eval.hpp:212-221); out [batch, output_count] fp32 or int8.
 * stream: a cudaStream_t (NULL = legacy default stream). */
kan_status kan_engine_forward(kan_engine* e, const float* x_dev, int64_t batch, void* out_dev,
                              void* stream);
/* Same on host buffers: H2D of x and D2H of the outputs are part of the call. */
kan_status kan_engine_forward_host(kan_engine* e, const float* x_host, int64_t batch,
                                   void* out_host, void* stream);
/* predict: argmax of the logits (first maximum wins, eval.hpp:268-272). */
kan_status kan_engine_predict(kan_engine* e, const float* x_dev, int64_t batch,
                              int32_t* labels_dev, void* stream);

/* evaluate_accuracy (eval.hpp:279-287): top-1 accuracy of predict against
 * int32 labels [batch] on the device (0 for an empty batch). */
kan_status kan_engine_evaluate_accuracy(kan_engine* e, const float* x_dev, const int32_t* labels_dev,
                                        int64_t batch, double* accuracy, void* stream);

/* Parity probes ------------------------------------------------------------ */
/* Lattice levels of fp32 activations under layer `layer`'s grid and lut_k
 * (spline-table mode: quantize_value on the grid bounds at bits_a). */
kan_status kan_engine_layer_levels(kan_engine* e, int layer, const float* x_dev, int64_t n,
                                   uint16_t* levels_dev, void* stream);
/* Raw int32 accumulators of one LUT layer given its input levels [batch, n_in]
 * (spline-table mode: acc_s = sum_i (table[i][j][level] - z_out), acc_b unused):
 * acc_s [batch, n_out] (spline part), acc_b [batch, n_out] (SiLU base part;
 * may be NULL). */
kan_status kan_engine_layer_accumulators(kan_engine* e, int layer, const uint16_t* levels_dev,
                                         int64_t batch, int32_t* acc_s_dev, int32_t* acc_b_dev,
                                         void* stream);
/* Training backward (train.hpp:84-160), fp32 ----------------------------- */
/* kan_linear_backward of linear KAN layer `layer` with its current
 * coefficients: x [batch, n_in] (the layer's inputs), dout [batch, n_out] ->
 * dcoeffs [n_in*(G+P), n_out] (reference row layout) and, if dinputs is not
 * NULL, dinputs [batch, n_in] (zero where clamp_to_domain moved x). */
kan_status kan_engine_linear_backward(kan_engine* e, int layer, const float* x_dev, int64_t batch,
                                      const float* dout_dev, float* dcoeffs_dev, float* dinputs_dev,
                                      void* stream);
/* conv layer backward (train.hpp:367-399): x [batch, c_in, H, W] (NCHW, the
 * layer's input), dout [batch, c_out, Ho, Wo] -> dcoeffs [c_in*K*K*(G+P), c_out]
 * and, if dinputs is not NULL, dinputs [batch, c_in, H, W] (col2im_add of the
 * patch gradients). */
kan_status kan_engine_conv_backward(kan_engine* e, int layer, const float* x_dev, int64_t batch,
                                    const float* dout_dev, float* dcoeffs_dev, float* dinputs_dev, void* stream);
/* maxpool2 (layers.hpp:193-205) forward and its backward (train.hpp:407-431:
 * the gradient goes to the first strict maximum of each window) on NCHW fp32
 * planes [planes, H, W]. */
kan_status kan_maxpool2_f32(const float* in_dev, int64_t planes, int H, int W, int window, float* out_dev,
                            void* stream);
kan_status kan_maxpool2_backward_f32(const float* in_dev, int64_t planes, int H, int W, int window,
                                     const float* dout_dev, float* din_dev, void* stream);
/* softmax_cross_entropy (train.hpp:139-160): per-row loss [batch] (the mean is
 * their average) and dL/dlogits [batch, n] = (softmax - onehot) / batch. */
/* One SGD-with-momentum update of a KAN layer's coefficients on the device:
 * v = momentum * v - lr * g; w += v (train.hpp:361-366, 401-404), in fp64 on a
 * device-resident master copy; the fp32 copies the forward and backward read
 * are refreshed in the same launch.  dcoeffs_dev is the gradient from
 * kan_engine_linear_backward / kan_engine_conv_backward ([n_in * (G+P), n_out]).
 * The engine must be configured in fp32 mode.  kan_engine_set_coeffs resets the
 * momentum; kan_engine_get_coeffs reads the current coefficients back. */
kan_status kan_engine_sgd_step(kan_engine* e, int layer, const float* dcoeffs_dev, double lr, double momentum,
                               void* stream);
kan_status kan_engine_get_coeffs(kan_engine* e, int layer, double* out, int64_t n);
kan_status kan_softmax_cross_entropy(const float* logits_dev, const int32_t* labels_dev, int64_t batch, int n,
                                     float* loss_rows_dev, float* dlogits_dev, void* stream);

/* Fake-quant calibrated activation policy (QuantConfig::ARangePolicy::kCalibrated,
 * EvalOptions::a_ranges, eval.hpp:43-68): ranges [n][2] = (lo, hi) per KAN layer,
 * as calibrate_activation_ranges returns them (eval.hpp:289-341); n = 0 restores
 * the grid-bound policy.  Takes effect at the next kan_engine_configure. */
kan_status kan_engine_set_activation_ranges(kan_engine* e, const double* ranges, int n);

/* Spline-table mode ------------------------------------------------------- */
/* Supply the tables of KAN layer `layer` (SplineTableSet, spline_table.hpp:19-34;
 * EvalOptions::tables, eval.hpp:41), e.g. read from a .kant container
 * (io.hpp:335-344), instead of building them from the coefficients at configure:
 * values [n_in][n_out][2^bits_a] (n_in = patch size for conv layers),
 * qp_d = {in_scale, out_scale}, qp_i = {in_zero_point, in_q_hi, out_zero_point,
 * out_q_hi}.  n = 0 clears them. */
kan_status kan_engine_set_spline_tables(kan_engine* e, int layer, const uint8_t* values, int64_t n,
                                        int bits_a, int h, const double* qp_d, const int64_t* qp_i);
/* Host copy of the configured tables of KAN layer `layer` in the reference
 * layout [n_in][n_out][2^bits_a] (SplineTableSet::values) and its quantizers
 * (as above).  Returns the entry count, or a negative status. */
int64_t kan_engine_spline_table(kan_engine* e, int layer, uint8_t* out, int64_t cap, double* qp_d,
                                int64_t* qp_i);

/* Host copy of the configured table (BsplineLut::entries). Returns entry count. */
int64_t kan_engine_lut(const kan_engine* e, uint8_t* out, int64_t cap);
/* Kernels launched by the most recent forward call. */
int kan_engine_last_launches(const kan_engine* e);
/* Per-layer kernel timing: when on, every forward brackets each KAN layer's
 * launch with CUDA events on the launching stream; kan_engine_layer_time_ms
 * waits for them and returns the accumulated device time and launch count of
 * layer `layer` since profiling was (re)enabled. */
kan_status kan_engine_set_profiling(kan_engine* e, int on);
kan_status kan_engine_layer_time_ms(kan_engine* e, int layer, double* total_ms, int64_t* count);
/* Tuning aid (active when the environment variable KAN_TIMELINE is set at
 * configure time): per-CTA %globaltimer stamps of layer `layer`'s most recent
 * launch, 8 per CTA (start, tables ready, first A stage, last A stage, TMEM
 * full, partials stored, done).  Returns the number of values (8 * CTAs). */
int64_t kan_engine_layer_timeline(kan_engine* e, int layer, unsigned long long* out, int64_t cap);

/* Tuning and debug switches (no reference counterpart; nothing is read from
 * the environment).  They take effect at the next kan_engine_configure, except
 * KAN_OPT_RECORD_PLAN, which applies to the following forwards.  Defaults are
 * the production choices; the others exist for A/B parity tests and tuning. */
typedef enum {
  KAN_OPT_NO_CONV3 = 1,           /* 1: 3x3 s1 convs take the general gather GEMM, not kan_conv3 */
  KAN_OPT_NO_IM2COL = 2,          /* 1: stem convs read the NHWC input instead of a level im2col */
  KAN_OPT_FORCE_BN = 3,           /* >0: cap the gather GEMM's N tile (multiple of 16) */
  KAN_OPT_TABLES = 4,             /* -1 auto, 0/1/2: force the shared-memory table variant */
  KAN_OPT_EPI_STAGE = 5,          /* 0: no smem-staged fp32 epilogue */
  KAN_OPT_CONV3_MC = 6,           /* CTAs per weight-multicast cluster in kan_conv3 (1 or 2) */
  KAN_OPT_LV_SIDECAR = 7,         /* 0: fp32-stored tensors carry no levels sidecar */
  KAN_OPT_LEVEL_PREPASS_MIN = 8,  /* fp32-input dense layers with >= this many activations get a level prepass */
  KAN_OPT_ST_PREPASS = 9,         /* 0: spline-table mode quantizes fp32 rows inside the gather kernel */
  KAN_OPT_ST_SLICES = 10,         /* >0: force the spline-table kernel's input slices per row */
  KAN_OPT_TIMELINE = 11,          /* 1: per-CTA phase stamps (kan_engine_layer_timeline) */
  KAN_OPT_FORCE_NACC1 = 12,       /* 1: one TMEM accumulator (deeper A ring) */
  KAN_OPT_RECORD_PLAN = 13,       /* 1: record each forward's launch plan (kan_engine_last_plan) */
  KAN_OPT_DBG_FLAGS = 14,         /* ablation bits; honoured only by a -DKAN_TUNING build */
  KAN_OPT_NO_CONVW = 15,          /* 1: 3x3 s1 convs skip the window-shared kan_convw kernel */
  KAN_OPT_CONVW_RINGS = 16,       /* kan_convw ring depths SA*100 + SB*10 + SX (0 = automatic) */
  KAN_OPT_CONVW_TR = 17,          /* kan_convw output rows per tile cap (0 = automatic) */
  KAN_OPT_CONVW_MC = 18,          /* kan_convw CTAs per weight-multicast cluster: 1, 2, 4 (0 = automatic) */
  KAN_OPT_CONVW_BN = 19,          /* kan_convw N tile cap, multiple of 16 (0 = automatic, 128) */
  KAN_OPT_NO_FUSE = 21,           /* 1: a small output layer always runs as its own launch (never inside the previous layer's kernel) */
  KAN_OPT_FUSE_PERSISTENT = 22,   /* 1: persistent (unsplit) launches also run a small output layer after each tile's epilogue */
  KAN_OPT_CONVW_NO_KYM = 23,      /* 1: kan_convw issues one MMA per (tap, output row) even where the ky-merged form applies */
  KAN_OPT_CONVW_DUAL = 24,        /* kan_convw second MMA-issuing warp (even / odd accumulators; single-commit layers without the ky-merged issue): -1 off, 1 on, 0 = automatic (on with two or more N tiles) */
  KAN_OPT_CONVW_LOCK = 20         /* kan_convw: one tcgen05.commit per K block releases the window slot and the weight slot (needs weight ring <= window ring): -1 off, 1 on, 0 = automatic (on for N tiles >= 128) */
} kan_option;
kan_status kan_engine_set_option(kan_engine* e, int option, int64_t value);
/* The launch plan of the most recent forward when KAN_OPT_RECORD_PLAN is on:
 * one line per kernel launch (kernel, KAN layer, epilogue kind, residual,
 * levels sidecar, N, N tile, K splits, mode).  Empty otherwise. */
const char* kan_engine_last_plan(const kan_engine* e);

/* Multi-GPU forward: one engine per device, contiguous batch
 * shards, no collective on the forward path; the logits of every shard land in
 * one buffer on engines[0]'s device (peer copies over NVLink).  The engines
 * must be configured identically from the same model (same output kind and
 * size); two engines may share a device.  Replaces the reference's chunk loop
 * of predict (eval.hpp:255-276) at box scale.
 *   x_shards[g]  device pointer on engines[g]'s device with rows
 *                [g*per, min(batch, (g+1)*per)) of the batch, per = ceil(batch/n)
 *                (kan_shard_rows); NULL for an empty shard
 *   out_dev0     [batch, output_count] on engines[0]'s device
 *   streams[g]   the stream each shard runs on (NULL = a per-engine stream);
 *                on return every stream's work is enqueued and streams[0]
 *                (or the legacy stream of device 0) waits for all shards */
kan_status kan_engine_forward_sharded(kan_engine* const* engines, int n_engines, const float* const* x_shards,
                                      int64_t batch, void* out_dev0, void* const* streams);
/* Same over host buffers (the serving call): x_host [batch, input_size] and
 * out_host [batch, output_count] (pinned memory gives asynchronous copies).
 * Each shard is copied to its device, run, and its logits copied back; the
 * call returns when every shard has landed in out_host. */
kan_status kan_engine_forward_sharded_host(kan_engine* const* engines, int n_engines, const float* x_host,
                                           int64_t batch, void* out_host);
/* Rows [*start, *stop) of shard g of n (contiguous, ceil(batch/n) rows each). */
void kan_shard_rows(int64_t batch, int g, int n, int64_t* start, int64_t* stop);

/* build_bspline_lut (lut.hpp:103-131) as a host utility. Returns entry count,
 * or -KAN_ERR_INVALID_ARGUMENT. */
int64_t kan_lut_build(int degree, int k, int h, uint8_t* out, int64_t cap);

/* Host utility: the lattice threshold table the GPU level kernel uses,
 * thr[n] = smallest fp32 x with level(x) >= n for n = 1..L (thr[0] = -inf,
 * thr[L+1] = NaN), level = ActivationLattice::quantize(clamp_to_domain(x))
 * (lut.hpp:44-47, grid.hpp:49-56).  `out` holds L+2 floats.  Returns L+2. */
int64_t kan_lattice_thresholds(int intervals, int degree, double lo, double hi, int k,
                               float* out, int64_t cap);

/* .kant model container (io.hpp:99-350) --------------------------------- */
/* Host-side reader: load_container (io.hpp:217-350).  Errors: missing file ->
 * KAN_ERR_IO, bad magic / unsupported version (named in the message) /
 * truncation -> KAN_ERR_FORMAT, payload CRC mismatch -> KAN_ERR_CHECKSUM.  On
 * error *out still holds a handle carrying the message (destroy it). */
typedef struct kan_container kan_container;
kan_status kan_container_load(const char* path, kan_container** out);
void kan_container_destroy(kan_container* c);
const char* kan_container_last_error(const kan_container* c);
/* the stored model in the descriptor schema kan_engine_create takes */
const char* kan_container_descriptor(const kan_container* c);
int kan_container_num_kan_layers(const kan_container* c);
/* coefficients of KAN layer `layer` (f32 in the file, widened to fp64), reference
 * row layout [n_in*(G+P), n_out]; returns the count */
int64_t kan_container_coeffs(const kan_container* c, int layer, double* out, int64_t cap);
/* the embedded BsplineLut entries (0 if none) and its degree / k / h */
int64_t kan_container_lut(const kan_container* c, uint8_t* out, int64_t cap, int* degree, int* k, int* h);
/* embedded SplineTableSets (one per KAN layer when present), as for
 * kan_engine_set_spline_tables */
int kan_container_num_spline_tables(const kan_container* c);
int64_t kan_container_spline_table(const kan_container* c, int t, uint8_t* out, int64_t cap, int* bits_a,
                                   int* h, double* qp_d, int64_t* qp_i);
/* save_container (io.hpp:108-211) of a descriptor-schema model: coeffs[i] =
 * KAN layer i's coefficients (stored as f32); optional LUT entries (lut == NULL:
 * none) and per-KAN-layer spline tables (st_values == NULL: none; qp arrays
 * [n_kan][2] / [n_kan][4] as above).  Byte-identical to the reference's file. */
kan_status kan_container_save(const char* path, const char* descriptor_json, const double* const* coeffs,
                              const uint8_t* lut, int64_t lut_n, int lut_k, int lut_h,
                              const uint8_t* const* st_values, int st_bits_a, int st_h, const double* st_qp_d,
                              const int64_t* st_qp_i);
const char* kan_container_save_error(void);
/* crc32 of io.hpp:31-45 (host utility) */
uint32_t kan_crc32(const uint8_t* data, size_t len);
/* load_model + engine: create from the container's model, set its coefficients,
 * its spline tables (if present) and its LUT (used by configure when lut_k /
 * lut_h match the stored table). */
kan_status kan_engine_load(const char* path, int device, kan_engine** out);

/* Host utility: the spline-table input level thresholds the GPU uses,
 * thr[n] = smallest fp32 x with quantize_value(x, in_qp) >= n for n = 1..2^bits_a-1
 * (thr[0] = -inf), in_qp = compute_quant_params(lo, hi, bits_a) (quant.hpp:33-54,
 * spline_table.hpp:51); thr[2^bits_a] = the smallest fp32 x whose llround
 * overflows (level 0 there, as for NaN, on the reference's x86-64 build).
 * Returns 2^bits_a + 1, or -KAN_ERR_INVALID_ARGUMENT. */
int64_t kan_spline_thresholds(double lo, double hi, int bits_a, float* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
