// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile directly from the
// reference's read-only include tree (-I/root/reference/proj/include) into
// oracle/_ref/libkantize_ref.so.  Nothing here re-implements the algorithm:
// every entry point forwards to the reference function named beside it, so
// the CPU oracle restatement (kan_oracle.c) and the CUDA engine can be
// checked against the reference itself, and bench.py --impl reference can
// time the reference's own CPU path.
// dataset.hpp (pulled in by eval.hpp) uses std::clamp/std::shuffle without
// including <algorithm>; provide it first rather than touching the reference.
#include <algorithm>
#include <random>

#include <kantize/eval.hpp>
#include <kantize/grid.hpp>
#include <kantize/io.hpp>
#include <kantize/layers.hpp>
#include <kantize/lut.hpp>
#include <kantize/quant.hpp>
#include <kantize/cost.hpp>
#include <kantize/spline_table.hpp>
#include <kantize/train.hpp>
#include <optional>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace kantize;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// compute_quant_params (quant.hpp:33-49)
int ref_quant_params(double a, double b, int bits, double* scale, int64_t* zp) try {
  const QuantParams qp = compute_quant_params(a, b, bits);
  *scale = qp.scale;
  *zp = qp.zero_point;
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// quantize_value (quant.hpp:51-54)
int64_t ref_quantize_value(double x, double a, double b, int bits) {
  return quantize_value(x, compute_quant_params(a, b, bits));
}

// GridSpec::clamp_to_domain + ActivationLattice::quantize (grid.hpp:49, lut.hpp:44)
int64_t ref_level_of(int G, int P, double lo, double hi, int k, double x) {
  const GridSpec g = build_grid(G, P, lo, hi);
  return ActivationLattice::of(g, k).quantize(g.clamp_to_domain(x));
}

void ref_levels_f32(int G, int P, double lo, double hi, int k, const float* x, int64_t n,
                    uint16_t* out) {
  const GridSpec g = build_grid(G, P, lo, hi);
  const ActivationLattice lat = ActivationLattice::of(g, k);
  for (int64_t i = 0; i < n; ++i)
    out[i] = static_cast<uint16_t>(lat.quantize(g.clamp_to_domain(static_cast<double>(x[i]))));
}

double ref_clamp(int G, int P, double lo, double hi, double x) {
  return build_grid(G, P, lo, hi).clamp_to_domain(x);
}

// build_bspline_lut (lut.hpp:103-131)
int ref_build_lut(int P, int k, int h, uint8_t* out, int64_t cap, int64_t* memory_bits) try {
  const BsplineLut lut = build_bspline_lut(P, k, h);
  if (static_cast<int64_t>(lut.entries.size()) > cap) return -1;
  std::copy(lut.entries.begin(), lut.entries.end(), out);
  if (memory_bits) *memory_bits = lut.memory_bits();
  return static_cast<int>(lut.entries.size());
} catch (const std::exception& e) {
  return fail(e);
}

// lut_basis_lookup (lut.hpp:136-160)
int ref_lut_lookup(int G, int P, double lo, double hi, int k, int h, int64_t a, uint8_t* vals,
                   int* start) try {
  const GridSpec g = build_grid(G, P, lo, hi);
  const BsplineLut lut = build_bspline_lut(P, k, h);
  const QuantizedBasis qb = lut_basis_lookup(a, g, lut);
  for (int r = 0; r < qb.count; ++r) vals[r] = qb.values[r];
  *start = qb.support_start;
  return qb.count;
} catch (const std::exception& e) {
  return fail(e);
}

// quantized_basis_reference (lut.hpp:164-180)
int ref_quantized_basis(int G, int P, double lo, double hi, int k, int h, int64_t a,
                        uint8_t* vals, int* start) try {
  const GridSpec g = build_grid(G, P, lo, hi);
  const ActivationLattice lat = ActivationLattice::of(g, k);
  const QuantizedBasis qb =
      quantized_basis_reference(a, g, lat, compute_quant_params(0.0, 1.0, h));
  for (int r = 0; r < qb.count; ++r) vals[r] = qb.values[r];
  *start = qb.support_start;
  return qb.count;
} catch (const std::exception& e) {
  return fail(e);
}

// cox_de_boor (grid.hpp:177-182)
int ref_cox_de_boor(int G, int P, double lo, double hi, double x, double* out) {
  const GridSpec g = build_grid(G, P, lo, hi);
  const BasisVector bv = cox_de_boor(x, g);
  std::copy(bv.values.begin(), bv.values.end(), out);
  return bv.support_start;
}

static KanLinearLayer make_linear(int G, int P, double lo, double hi, int n_in, int n_out,
                                  const double* coeffs) {
  KanLinearLayer l = KanLinearLayer::zeros(n_in, n_out, build_grid(G, P, lo, hi));
  std::copy(coeffs, coeffs + l.coeffs.size(), l.coeffs.flat().begin());
  return l;
}

static Matrix make_matrix(int64_t rows, int64_t cols, const double* src) {
  Matrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  std::copy(src, src + rows * cols, m.flat().begin());
  return m;
}

// kan_linear_forward with RecursiveBasis (layers.hpp:118-121)
int ref_linear_forward(int G, int P, double lo, double hi, int64_t M, int n_in, int n_out,
                       const double* acts, const double* coeffs, double* out) try {
  const KanLinearLayer l = make_linear(G, P, lo, hi, n_in, n_out, coeffs);
  const Matrix r = kan_linear_forward(make_matrix(M, n_in, acts), l);
  std::copy(r.flat().begin(), r.flat().end(), out);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// tabulated_kan_forward (lut.hpp:217-231)
int ref_lut_forward(int G, int P, double lo, double hi, int k, int h, int bits_w, int64_t M,
                    int n_in, int n_out, const double* acts, const double* coeffs,
                    double* out) try {
  const KanLinearLayer l = make_linear(G, P, lo, hi, n_in, n_out, coeffs);
  const BsplineLut lut = build_bspline_lut(P, k, h);
  const Matrix r = tabulated_kan_forward(make_matrix(M, n_in, acts), l, lut, bits_w);
  std::copy(r.flat().begin(), r.flat().end(), out);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// kan_linear_forward with LatticeQuantBasis (lut.hpp:200-213)
int ref_latticequant_forward(int G, int P, double lo, double hi, int k, int h, int64_t M,
                             int n_in, int n_out, const double* acts, const double* coeffs,
                             double* out) try {
  const KanLinearLayer l = make_linear(G, P, lo, hi, n_in, n_out, coeffs);
  const ActivationLattice lat = ActivationLattice::of(l.grid, k);
  const Matrix r = kan_linear_forward(make_matrix(M, n_in, acts), l,
                                      LatticeQuantBasis{&l.grid, lat,
                                                        compute_quant_params(0.0, 1.0, h)});
  std::copy(r.flat().begin(), r.flat().end(), out);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// im2col (layers.hpp:126-154)
int ref_im2col(const double* in, int C, int H, int W, int kernel, int stride, int padding,
               double* out) try {
  Tensor3 t(C, H, W);
  std::copy(in, in + t.size(), t.data.begin());
  const Matrix m = im2col(t, kernel, stride, padding);
  std::copy(m.flat().begin(), m.flat().end(), out);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// convkan_forward (layers.hpp:162-190); mode 0 = RecursiveBasis, 1 = LUT
// (LutBasis over fake-quantized weights as forward_conv does in bspline-lut
// mode, eval.hpp:185-188 + eval.hpp:116).
int ref_conv_forward(int G, int P, double lo, double hi, int mode, int k, int h, int bits_w,
                     int C, int H, int W, int c_out, int kernel, int stride, int padding,
                     const double* in, const double* coeffs, double* out) try {
  const GridSpec g = build_grid(G, P, lo, hi);
  ConvKanLayer conv = ConvKanLayer::zeros(C, c_out, kernel, stride, padding, g);
  std::copy(coeffs, coeffs + conv.coeffs.size(), conv.coeffs.flat().begin());
  Tensor3 t(C, H, W);
  std::copy(in, in + t.size(), t.data.begin());
  Tensor3 r;
  if (mode == 0) {
    r = convkan_forward(t, conv);
  } else {
    const BsplineLut lut = build_bspline_lut(P, k, h);
    conv.coeffs = detail::maybe_fake_quant_weights(conv.coeffs, bits_w);
    LutBasis basis{&conv.grid, &lut, ActivationLattice::of(conv.grid, k)};
    r = convkan_forward(t, conv, basis);
  }
  std::copy(r.data.begin(), r.data.end(), out);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// build_spline_tables (spline_table.hpp:87-95) for a linear layer (kernel == 0)
// or a conv layer (c_in = n_in, c_out = n_out, kernel/stride/padding); values
// [table_count * 2^bits_a]; qp_d = {in_scale, out_scale}; qp_i = {in_zp,
// in_qhi, out_zp, out_qhi}.  Returns stored_bits(), or -1.
int64_t ref_spline_tables(int G, int P, double lo, double hi, int n_in, int n_out, int kernel,
                          int stride, int padding, const double* coeffs, int bits_a, int h,
                          uint8_t* values, int64_t cap, double* qp_d, int64_t* qp_i) try {
  const GridSpec g = build_grid(G, P, lo, hi);
  SplineTableSet set;
  if (kernel == 0) {
    KanLinearLayer l = KanLinearLayer::zeros(n_in, n_out, g);
    std::copy(coeffs, coeffs + l.coeffs.size(), l.coeffs.flat().begin());
    set = build_spline_tables(l, bits_a, h);
  } else {
    ConvKanLayer c = ConvKanLayer::zeros(n_in, n_out, kernel, stride, padding, g);
    std::copy(coeffs, coeffs + c.coeffs.size(), c.coeffs.flat().begin());
    set = build_spline_tables(c, bits_a, h);
  }
  if (static_cast<int64_t>(set.values.size()) > cap) {
    g_err = "ref_spline_tables: capacity";
    return -1;
  }
  std::copy(set.values.begin(), set.values.end(), values);
  qp_d[0] = set.in_qp.scale;
  qp_d[1] = set.out_qp.scale;
  qp_i[0] = set.in_qp.zero_point;
  qp_i[1] = set.in_qp.q_hi;
  qp_i[2] = set.out_qp.zero_point;
  qp_i[3] = set.out_qp.q_hi;
  return set.stored_bits();
} catch (const std::exception& e) {
  return fail(e);
}

// spline_table_forward (spline_table.hpp:90-107) over a table set rebuilt
// from its parts (values [n_in][n_out][2^bits_a], quantizers as above)
int ref_spline_table_forward(int n_in, int n_out, int bits_a, int h, const uint8_t* values,
                             const double* qp_d, const int64_t* qp_i, int64_t M,
                             const double* acts, double* out) try {
  SplineTableSet set;
  set.n_in = n_in;
  set.n_out = n_out;
  set.bits_a = bits_a;
  set.value_bits = h;
  set.in_qp = compute_quant_params(-1.0, 1.0, bits_a);
  set.in_qp.scale = qp_d[0];
  set.in_qp.zero_point = qp_i[0];
  set.in_qp.q_hi = qp_i[1];
  set.out_qp = compute_quant_params(-1.0, 1.0, h);
  set.out_qp.scale = qp_d[1];
  set.out_qp.zero_point = qp_i[2];
  set.out_qp.q_hi = qp_i[3];
  set.values.assign(values, values + set.table_count() * set.entries_per_table());
  const Matrix r = spline_table_forward(make_matrix(M, n_in, acts), set);
  std::copy(r.flat().begin(), r.flat().end(), out);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// cost.hpp:68-74 mul_counts_layer().matmul via a descriptor (algorithmic work)
int ref_validate_descriptor(const char* json_text) try {
  const Model m = model_from_descriptor(nlohmann::json::parse(json_text));
  return static_cast<int>(m.layers.size());
} catch (const std::exception& e) {
  return fail(e);
}

// model_forward / predict (eval.hpp:200-276) over a descriptor-built model
// (io.hpp:357-386).  coeff_ptrs[i] = coefficients of the i-th KAN layer.
// mode: 0 fp32 (EvalMode::kFp32), 1 fake-quant (EvalMode::kFakeQuant; bits_w,
// bits_a = k, bits_b = h), 2 bspline-lut (EvalMode::kBsplineLut),
// 3 spline-table (EvalMode::kSplineTable; bits_a = k, value bits = h).
// The batch is sharded over `threads` std::threads in chunks of `chunk`
// rows (the forward is reentrant).
int ref_model_forward(const char* json_text, const double* const* coeff_ptrs, int mode, int k,
                      int h, int bits_w, int64_t M, int64_t D, const double* inputs,
                      int64_t n_out, double* out, int threads, int64_t chunk) try {
  Model model = model_from_descriptor(nlohmann::json::parse(json_text));
  int li = 0;
  for (auto& layer : model.layers) {
    if (auto* lin = std::get_if<KanLinearLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + lin->coeffs.size(), lin->coeffs.flat().begin());
      ++li;
    } else if (auto* conv = std::get_if<ConvKanLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + conv->coeffs.size(),
                conv->coeffs.flat().begin());
      ++li;
    }
  }
  const BsplineLut lut = build_bspline_lut(model.grid().degree(), mode == 2 ? k : 8, mode == 2 ? h : 8);
  // spline-table mode: one table set per KAN layer at (bits_a = k, h), as
  // run_sweep builds them (sweep.hpp:239-256)
  std::vector<SplineTableSet> tables;
  if (mode == 3)
    for (const auto& layer : model.layers) {
      if (const auto* lin = std::get_if<KanLinearLayer>(&layer))
        tables.push_back(build_spline_tables(*lin, k, h));
      else if (const auto* conv = std::get_if<ConvKanLayer>(&layer))
        tables.push_back(build_spline_tables(*conv, k, h));
    }
  EvalOptions opts;
  opts.mode = mode == 2 ? EvalMode::kBsplineLut
                       : (mode == 3 ? EvalMode::kSplineTable : (mode == 1 ? EvalMode::kFakeQuant : EvalMode::kFp32));
  opts.qcfg.bits_w = (mode == 2 || mode == 1) ? bits_w : kPassthroughBits;
  if (mode == 1) {  // fake-quant: bits_a = k, bits_b = h (sweep.hpp:262-266), grid-bound ranges
    opts.qcfg.bits_a = k;
    opts.qcfg.bits_b = h;
  }
  opts.lut = &lut;
  opts.tables = &tables;
  if (threads < 1) threads = 1;
  if (chunk < 1) chunk = 256;
  std::vector<std::thread> pool;
  std::vector<std::string> errs(static_cast<std::size_t>(threads));
  const int64_t per = (M + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      try {
        const int64_t r0 = t * per, r1 = std::min(M, r0 + per);
        for (int64_t s = r0; s < r1; s += chunk) {
          const int64_t rows = std::min(chunk, r1 - s);
          const Matrix logits = model_forward(model, make_matrix(rows, D, inputs + s * D), opts);
          std::copy(logits.flat().begin(), logits.flat().end(), out + s * n_out);
        }
      } catch (const std::exception& e) {
        errs[static_cast<std::size_t>(t)] = e.what();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (!e.empty()) {
      g_err = e;
      return -1;
    }
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// spline-table model_forward with the tables built ONCE up front (as run_sweep
// does, sweep.hpp:239-256, and as a caller passing EvalOptions::tables does);
// the batch runs `reps` times sharded over `threads` std::threads in `chunk`
// rows; *seconds = wall time of the forwards alone (the CPU baseline of the
// spline-table bench lines).
int ref_st_model_forward(const char* json_text, const double* const* coeff_ptrs, int bits_a, int h,
                         int64_t M, int64_t D, const double* inputs, int64_t n_out, double* out,
                         int threads, int64_t chunk, int reps, double* seconds) try {
  Model model = model_from_descriptor(nlohmann::json::parse(json_text));
  int li = 0;
  std::vector<SplineTableSet> tables;
  for (auto& layer : model.layers) {
    if (auto* lin = std::get_if<KanLinearLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + lin->coeffs.size(), lin->coeffs.flat().begin());
      tables.push_back(build_spline_tables(*lin, bits_a, h));
      ++li;
    } else if (auto* conv = std::get_if<ConvKanLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + conv->coeffs.size(), conv->coeffs.flat().begin());
      tables.push_back(build_spline_tables(*conv, bits_a, h));
      ++li;
    }
  }
  EvalOptions opts;
  opts.mode = EvalMode::kSplineTable;
  opts.tables = &tables;
  if (threads < 1) threads = 1;
  if (chunk < 1) chunk = 256;
  if (reps < 1) reps = 1;
  std::vector<std::string> errs(static_cast<std::size_t>(threads));
  const int64_t per = (M + threads - 1) / threads;
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          const int64_t r0 = t * per, r1 = std::min(M, r0 + per);
          for (int64_t s = r0; s < r1; s += chunk) {
            const int64_t rows = std::min(chunk, r1 - s);
            const Matrix logits = model_forward(model, make_matrix(rows, D, inputs + s * D), opts);
            std::copy(logits.flat().begin(), logits.flat().end(), out + s * n_out);
          }
        } catch (const std::exception& e) {
          errs[static_cast<std::size_t>(t)] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
  }
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (auto& e : errs)
    if (!e.empty()) {
      g_err = e;
      return -1;
    }
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// save_container (io.hpp:108-211) of a descriptor-built model with its
// coefficients; lut_k > 0 adds build_bspline_lut(P, lut_k, lut_h); st_bits_a > 0
// adds build_spline_tables(layer, st_bits_a, st_h) for every KAN layer.
int ref_save_container(const char* json_text, const double* const* coeff_ptrs, int lut_k, int lut_h,
                       int st_bits_a, int st_h, const char* path) try {
  Model model = model_from_descriptor(nlohmann::json::parse(json_text));
  int li = 0;
  std::vector<SplineTableSet> tables;
  for (auto& layer : model.layers) {
    if (auto* lin = std::get_if<KanLinearLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + lin->coeffs.size(), lin->coeffs.flat().begin());
      if (st_bits_a > 0) tables.push_back(build_spline_tables(*lin, st_bits_a, st_h));
      ++li;
    } else if (auto* conv = std::get_if<ConvKanLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + conv->coeffs.size(), conv->coeffs.flat().begin());
      if (st_bits_a > 0) tables.push_back(build_spline_tables(*conv, st_bits_a, st_h));
      ++li;
    }
  }
  std::optional<BsplineLut> lut;
  if (lut_k > 0) lut = build_bspline_lut(model.grid().degree(), lut_k, lut_h);
  save_container(model, path, lut ? &*lut : nullptr, st_bits_a > 0 ? &tables : nullptr);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// load_container (io.hpp:217-350): number of layers, or -6 io_error,
// -7 format_error, -8 checksum_error, -1 other
int ref_load_container(const char* path) {
  try {
    return static_cast<int>(load_container(path).model.layers.size());
  } catch (const io_error& e) {
    g_err = e.what();
    return -6;
  } catch (const format_error& e) {
    g_err = e.what();
    return -7;
  } catch (const checksum_error& e) {
    g_err = e.what();
    return -8;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// calibrate_activation_ranges (eval.hpp:289-341) of a descriptor-built model:
// ranges [n_kan][2] (lo, hi)
int ref_calibrate_ranges(const char* json_text, const double* const* coeff_ptrs, int64_t M, int64_t D,
                         const double* inputs, double* ranges) try {
  Model model = model_from_descriptor(nlohmann::json::parse(json_text));
  int li = 0;
  for (auto& layer : model.layers) {
    if (auto* lin = std::get_if<KanLinearLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + lin->coeffs.size(), lin->coeffs.flat().begin());
      ++li;
    } else if (auto* conv = std::get_if<ConvKanLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + conv->coeffs.size(), conv->coeffs.flat().begin());
      ++li;
    }
  }
  const auto r = calibrate_activation_ranges(model, make_matrix(M, D, inputs));
  for (std::size_t i = 0; i < r.size(); ++i) {
    ranges[2 * i] = r[i].first;
    ranges[2 * i + 1] = r[i].second;
  }
  return static_cast<int>(r.size());
} catch (const std::exception& e) {
  return fail(e);
}

// model_forward in fake-quant mode with the calibrated activation policy
// (QuantConfig::ARangePolicy::kCalibrated, eval.hpp:55-68): ranges [n_kan][2]
int ref_fakequant_calibrated_forward(const char* json_text, const double* const* coeff_ptrs, int bits_w,
                                     int bits_a, int bits_b, const double* ranges, int64_t M, int64_t D,
                                     const double* inputs, int64_t n_out, double* out) try {
  Model model = model_from_descriptor(nlohmann::json::parse(json_text));
  int li = 0;
  for (auto& layer : model.layers) {
    if (auto* lin = std::get_if<KanLinearLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + lin->coeffs.size(), lin->coeffs.flat().begin());
      ++li;
    } else if (auto* conv = std::get_if<ConvKanLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + conv->coeffs.size(), conv->coeffs.flat().begin());
      ++li;
    }
  }
  EvalOptions opts;
  opts.mode = EvalMode::kFakeQuant;
  opts.qcfg.bits_w = bits_w;
  opts.qcfg.bits_a = bits_a;
  opts.qcfg.bits_b = bits_b;
  opts.qcfg.a_range_policy = QuantConfig::ARangePolicy::kCalibrated;
  for (int i = 0; i < li; ++i) opts.a_ranges.emplace_back(ranges[2 * i], ranges[2 * i + 1]);
  const Matrix r = model_forward(model, make_matrix(M, D, inputs), opts);
  if (static_cast<int64_t>(r.cols()) != n_out) {
    g_err = "ref_fakequant_calibrated_forward: output width";
    return -1;
  }
  std::copy(r.flat().begin(), r.flat().end(), out);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// kan_linear_backward (train.hpp:131-136): dcoeffs [n_in*nb, n_out], dinputs [M, n_in]
int ref_linear_backward(int G, int P, double lo, double hi, int64_t M, int n_in, int n_out, const double* acts,
                        const double* coeffs, const double* dout, double* dcoeffs, double* dinputs) try {
  const KanLinearLayer l = make_linear(G, P, lo, hi, n_in, n_out, coeffs);
  const LayerGrads g = kan_linear_backward(make_matrix(M, n_in, acts), l, make_matrix(M, n_out, dout));
  std::copy(g.d_coeffs.flat().begin(), g.d_coeffs.flat().end(), dcoeffs);
  std::copy(g.d_inputs.flat().begin(), g.d_inputs.flat().end(), dinputs);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// softmax_cross_entropy (train.hpp:139-160): returns the mean loss in *loss
int ref_softmax_ce(int64_t M, int n, const double* logits, const int32_t* labels, double* dlogits,
                   double* loss) try {
  std::vector<int> lab(labels, labels + M);
  Matrix d;
  *loss = softmax_cross_entropy(make_matrix(M, n, logits), lab, d);
  std::copy(d.flat().begin(), d.flat().end(), dlogits);
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// train (train.hpp:247-462) of a descriptor-built model on (inputs, labels):
// SGD with momentum, `epochs` epochs of `batch` rows; coefficients updated in
// place in coeff_out (same layout as coeff_ptrs); returns the last epoch loss
// in *loss
int ref_train(const char* json_text, const double* const* coeff_ptrs, double* const* coeff_out, int64_t M,
              int64_t D, const double* inputs, const int32_t* labels, double lr, double momentum, int epochs,
              int batch, uint64_t seed, double* loss) try {
  Model model = model_from_descriptor(nlohmann::json::parse(json_text));
  int li = 0;
  for (auto& layer : model.layers) {
    if (auto* lin = std::get_if<KanLinearLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + lin->coeffs.size(), lin->coeffs.flat().begin());
      ++li;
    } else if (auto* conv = std::get_if<ConvKanLayer>(&layer)) {
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + conv->coeffs.size(), conv->coeffs.flat().begin());
      ++li;
    }
  }
  Dataset ds;
  ds.inputs = make_matrix(M, D, inputs);
  ds.labels.assign(labels, labels + M);
  TrainConfig cfg;
  cfg.lr = lr;
  cfg.momentum = momentum;
  cfg.epochs = epochs;
  cfg.batch = batch;
  cfg.seed = seed;
  const TrainResult r = train(model, ds, cfg);
  *loss = r.epoch_losses.empty() ? 0.0 : r.epoch_losses.back();
  li = 0;
  for (auto& layer : model.layers) {
    if (auto* lin = std::get_if<KanLinearLayer>(&layer)) {
      std::copy(lin->coeffs.flat().begin(), lin->coeffs.flat().end(), coeff_out[li++]);
    } else if (auto* conv = std::get_if<ConvKanLayer>(&layer)) {
      std::copy(conv->coeffs.flat().begin(), conv->coeffs.flat().end(), coeff_out[li++]);
    }
  }
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

// Harness composition for descriptors the reference cannot express (the
// engine's additive extension: named tensors id / input_from / residual,
// global_avgpool, "conv_output": "floor"), built ONLY from reference
// functions: convkan_forward with LutBasis over maybe_fake_quant_weights
// (eval.hpp:70-76, 185-188), kan_linear_forward, maxpool2, flatten.  Residual
// adds and the global average pool are harness fp64 loops; a stride that does
// not divide the padded span runs the reference on the input zero-extended at
// the bottom/right and crops (SURVEY.md 8(c) stride-2 recipe).  Used as the
// CPU baseline for ResKAN18 (C5); samples are sharded over std::threads.
int ref_graph_forward(const char* json_text, const double* const* coeff_ptrs, int k, int h,
                      int bits_w, int64_t M, const double* inputs, int64_t n_out, double* out,
                      int threads) try {
  const nlohmann::json j = nlohmann::json::parse(json_text);
  const GridSpec grid = build_grid(j["grid"]["intervals"].get<int>(), j["grid"]["degree"].get<int>(),
                                   j.contains("domain") ? j["domain"][0].get<double>() : -1.0,
                                   j.contains("domain") ? j["domain"][1].get<double>() : 1.0);
  const BsplineLut lut = build_bspline_lut(grid.degree(), k, h);
  const LutBasis basis{&grid, &lut, ActivationLattice::of(grid, k)};
  const std::vector<int> in_shape = j["input"].get<std::vector<int>>();
  struct L {
    std::string type, id, from, res;
    ConvKanLayer conv;
    KanLinearLayer lin;
    int window = 2;
  };
  std::vector<L> layers;
  int li = 0;
  for (const auto& jl : j["layers"]) {
    L l;
    l.type = jl["type"].get<std::string>();
    if (jl.contains("id")) l.id = jl["id"].get<std::string>();
    if (jl.contains("input_from")) l.from = jl["input_from"].get<std::string>();
    if (jl.contains("residual")) l.res = jl["residual"].get<std::string>();
    if (l.type == "conv") {
      l.conv = ConvKanLayer::zeros(jl["c_in"].get<int>(), jl["c_out"].get<int>(), jl["kernel"].get<int>(),
                                   jl.value("stride", 1), jl.value("padding", 0), grid);
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + l.conv.coeffs.size(), l.conv.coeffs.flat().begin());
      l.conv.coeffs = detail::maybe_fake_quant_weights(l.conv.coeffs, bits_w);
      ++li;
    } else if (l.type == "linear") {
      l.lin = KanLinearLayer::zeros(jl["n_in"].get<int>(), jl["n_out"].get<int>(), grid);
      std::copy(coeff_ptrs[li], coeff_ptrs[li] + l.lin.coeffs.size(), l.lin.coeffs.flat().begin());
      l.lin.coeffs = detail::maybe_fake_quant_weights(l.lin.coeffs, bits_w);
      ++li;
    } else if (l.type == "maxpool") {
      l.window = jl.value("window", 2);
    }
    layers.push_back(std::move(l));
  }
  const int64_t D = in_shape.size() == 3 ? int64_t{in_shape[0]} * in_shape[1] * in_shape[2] : in_shape[0];
  // a value is either an image (Tensor3) or a flat vector
  struct V {
    bool img = false;
    Tensor3 t;
    std::vector<double> v;
  };
  auto run_sample = [&](const double* x, double* y) {
    std::vector<std::pair<std::string, V>> named;
    V cur;
    if (in_shape.size() == 3) {
      cur.img = true;
      cur.t = Tensor3(in_shape[0], in_shape[1], in_shape[2]);
      std::copy(x, x + D, cur.t.data.begin());
    } else {
      cur.v.assign(x, x + D);
    }
    named.push_back({"input", cur});
    auto get = [&](const std::string& n) -> const V& {
      for (auto& kv : named)
        if (kv.first == n) return kv.second;
      throw std::invalid_argument("unknown tensor " + n);
    };
    for (const auto& l : layers) {
      V src = l.from.empty() ? cur : get(l.from);
      V o;
      if (l.type == "conv") {
        const ConvKanLayer& c = l.conv;
        Tensor3 t = src.t;
        const int ho = (t.height + 2 * c.padding - c.kernel) / c.stride + 1;
        const int wo = (t.width + 2 * c.padding - c.kernel) / c.stride + 1;
        int eh = t.height, ew = t.width;
        while ((eh + 2 * c.padding - c.kernel) % c.stride) ++eh;
        while ((ew + 2 * c.padding - c.kernel) % c.stride) ++ew;
        if (eh != t.height || ew != t.width) {
          Tensor3 ext(t.channels, eh, ew);
          for (int ch = 0; ch < t.channels; ++ch)
            for (int yy = 0; yy < t.height; ++yy)
              for (int xx = 0; xx < t.width; ++xx) ext.at(ch, yy, xx) = t.at(ch, yy, xx);
          t = std::move(ext);
        }
        Tensor3 r = convkan_forward(t, c, basis);
        o.img = true;
        o.t = Tensor3(r.channels, ho, wo);
        for (int ch = 0; ch < r.channels; ++ch)
          for (int yy = 0; yy < ho; ++yy)
            for (int xx = 0; xx < wo; ++xx) o.t.at(ch, yy, xx) = r.at(ch, yy, xx);
      } else if (l.type == "linear") {
        const std::vector<double>& in = src.img ? src.t.data : src.v;
        const Matrix r = kan_linear_forward(make_matrix(1, static_cast<int64_t>(in.size()), in.data()),
                                            l.lin, basis);
        o.v.assign(r.flat().begin(), r.flat().end());
      } else if (l.type == "maxpool") {
        o.img = true;
        o.t = maxpool2(src.t, l.window);
      } else if (l.type == "flatten") {
        o.v = flatten(src.t);
      } else if (l.type == "global_avgpool") {
        const int hw = src.t.height * src.t.width;
        o.v.assign(static_cast<std::size_t>(src.t.channels), 0.0);
        for (int ch = 0; ch < src.t.channels; ++ch) {
          double acc = 0.0;
          for (int q = 0; q < hw; ++q) acc += src.t.data[static_cast<std::size_t>(ch) * hw + q];
          o.v[static_cast<std::size_t>(ch)] = acc / hw;
        }
      } else {
        throw std::invalid_argument("unknown layer type " + l.type);
      }
      if (!l.res.empty()) {
        const V& r = get(l.res);
        std::vector<double>& dst = o.img ? o.t.data : o.v;
        const std::vector<double>& add = r.img ? r.t.data : r.v;
        for (std::size_t q = 0; q < dst.size(); ++q) dst[q] += add[q];
      }
      if (!l.id.empty()) named.push_back({l.id, o});
      cur = std::move(o);
    }
    const std::vector<double>& res = cur.img ? cur.t.data : cur.v;
    std::copy(res.begin(), res.begin() + n_out, y);
  };
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  std::vector<std::string> errs(static_cast<std::size_t>(threads));
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      try {
        for (int64_t s = t; s < M; s += threads) run_sample(inputs + s * D, out + s * n_out);
      } catch (const std::exception& e) {
        errs[static_cast<std::size_t>(t)] = e.what();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (!e.empty()) {
      g_err = e;
      return -1;
    }
  return 0;
} catch (const std::exception& e) {
  return fail(e);
}

}  // extern "C"
