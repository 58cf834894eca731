// rsparse_b200.hpp -- the C++ adapter a reference maintainer adds to
// rsparse (/root/reference/proj/core) to run its operator on a B200:
// rsparse::b200::Layer wraps a DecomposedLayer (layer.hpp:38-48) resident in
// HBM behind the C ABI of include/rsparse_b200.h, with the same contract as
// rsparse::forward(const DecomposedLayer&, std::span<const double>)
// (layer.hpp:75): a fresh std::vector<double> of m_out outputs, usage_error
// on a length mismatch (layer.cpp:96-99).  Errors map back onto the
// reference's exception taxonomy (errors.hpp:8-22).
//
// Compiled and run by tests/test_integration.py against the reference's own
// headers and sources (integration/Makefile).
#pragma once

#include <cstddef>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "rsparse/errors.hpp"
#include "rsparse/layer.hpp"
#include "rsparse_b200.h"

namespace rsparse::b200 {

inline void check(rsp_status st) {
  if (st == RSP_OK) return;
  const std::string msg = rsp_last_error();
  if (st == RSP_E_USAGE) throw usage_error(msg);
  if (st == RSP_E_NUMERIC) throw numeric_error(msg);
  if (st == RSP_E_IO) throw io_error(msg);
  throw std::runtime_error(msg);
}

// A DecomposedLayer resident in B200 HBM (bf16 weights by default).
class Layer {
 public:
  explicit Layer(const DecomposedLayer& L, rsp_dtype weights = RSP_BF16, int device = 0) {
    rsp_linear_desc d{};
    d.m_in = static_cast<uint32_t>(L.m_in);
    d.m_out = static_cast<uint32_t>(L.m_out);
    d.rank = static_cast<uint32_t>(L.plan.rank);
    d.keep_fraction = L.plan.keep_fraction;
    d.k_override = -1;
    d.weight_dtype = weights;
    d.src_dtype = RSP_F64;
    d.src_memory = RSP_MEM_HOST;
    d.w_layout = RSP_W_COL_MAJOR;  // w_cols.data: data[j * m_out + i] == W(i, j)
    d.w = L.w_cols.data.data();
    d.a_r = L.plan.rank ? L.a_r.data() : nullptr;
    d.b_r = L.plan.rank ? L.b_r.data() : nullptr;
    d.device = device;
    d.shard_count = 1;
    rsp_linear* h = nullptr;
    check(rsp_linear_create(&d, &h));
    h_.reset(h);
    if (!L.selected_components.empty()) {
      std::vector<uint32_t> comps(L.selected_components.begin(), L.selected_components.end());
      check(rsp_linear_set_components(h_.get(), comps.data(), static_cast<uint32_t>(comps.size())));
    }
    check(rsp_linear_info_get(h_.get(), &info_));
  }

  std::size_t m_in() const { return info_.m_in; }
  std::size_t m_out() const { return info_.m_out; }

  // rsparse::forward(layer, x) (layer.cpp:95-123), computed on the device.
  std::vector<double> forward(std::span<const double> x) const {
    if (x.size() != info_.m_in)
      throw usage_error("forward: input length " + std::to_string(x.size()) + " does not match m_in " +
                        std::to_string(info_.m_in));
    std::vector<float> xf(x.begin(), x.end());
    std::vector<double> y(info_.m_out);
    check(rsp_linear_forward_host(h_.get(), xf.data(), RSP_F32, y.data(), RSP_F64, 1));
    return y;
  }

  // B independent forwards: xs row-major B x m_in.
  std::vector<double> forward_batch(std::span<const double> xs, std::size_t batch) const {
    if (xs.size() != batch * info_.m_in) throw usage_error("forward_batch: input size mismatch");
    std::vector<float> xf(xs.begin(), xs.end());
    std::vector<double> y(batch * info_.m_out);
    check(rsp_linear_forward_host(h_.get(), xf.data(), RSP_F32, y.data(), RSP_F64, static_cast<uint32_t>(batch)));
    return y;
  }

  // rsparse::io_cost(layer) (layer.cpp:125-140) plus the kernel's own bytes.
  rsp_io_report io_cost() const {
    rsp_io_report r{};
    check(rsp_linear_io_cost(h_.get(), &r));
    return r;
  }

  const rsp_linear* handle() const { return h_.get(); }

 private:
  struct Del {
    void operator()(rsp_linear* p) const { rsp_linear_destroy(p); }
  };
  std::unique_ptr<rsp_linear, Del> h_;
  rsp_linear_info info_{};
};

}  // namespace rsparse::b200
