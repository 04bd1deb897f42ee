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

#include <algorithm>
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

// cost.hpp:68-74 mul_counts_layer().matmul via a descriptor (algorithmic work)
int ref_validate_descriptor(const char* json_text) try {
  const Model m = model_from_descriptor(nlohmann::json::parse(json_text));
  return static_cast<int>(m.layers.size());
} catch (const std::exception& e) {
  return fail(e);
}

// model_forward / predict (eval.hpp:200-276) over a descriptor-built model
// (io.hpp:357-386).  coeff_ptrs[i] = coefficients of the i-th KAN layer.
// mode: 0 fp32 (EvalMode::kFp32), 2 bspline-lut (EvalMode::kBsplineLut).
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
  const BsplineLut lut = build_bspline_lut(model.grid().degree(), k, h);
  EvalOptions opts;
  opts.mode = mode == 2 ? EvalMode::kBsplineLut : EvalMode::kFp32;
  opts.qcfg.bits_w = mode == 2 ? bits_w : kPassthroughBits;
  opts.lut = &lut;
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

}  // extern "C"
