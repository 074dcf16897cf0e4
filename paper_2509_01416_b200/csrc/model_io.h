// model_io.h — trained-operator model files (SPEC.md:349-357 save_model/load_model, :373 format).
//
// The reference fixes the container, not the record: a little-endian stream with a running
// FNV-1a-64 digest and the digest appended at the end (proj/core/include/snop/binary_io.hpp:12-62,
// src/binary_io.cpp:12-17,73-83,136-141). The record laid into it (format version 1):
//
//   string magic "SNOP-MODEL"      (u32 length + bytes, as BinaryWriter::write_string)
//   u32    version = 1
//   string arch "deeponet" | "fno"
//   f64 grid.length_cm, u64 grid.n_cells, f64 p*.sigma_t, f64 p*.sigma_s0, u32 activation
//   deeponet: u32 nb, u64 branch_sizes[nb], u32 nt, u64 trunk_sizes[nt], u8 has_bias0, f64 bias0
//   fno:      u64 width, u64 modes, u64 layers, u64 hidden
//   u64 n_params, f64 params[n_params]   (deeponet: branch then trunk, each layer W[out][in] then b;
//                                          fno: lift W,b; per layer R_re,R_im,W,b; P1 W,b; P2 W,b)
//   u64 FNV-1a-64 digest of every preceding byte
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/snop_cuda.h"

namespace snop_impl {

struct ModelFile {
  int arch = 0;  // SNOP_ARCH_DEEPONET / SNOP_ARCH_FNO
  snop_grid grid{};
  double tstar = 1.0, sstar = 0.5;
  int act = 1;
  std::vector<int32_t> bs, ts;  // DeepONet layer sizes
  bool has_bias0 = false;
  float bias0 = 0.f;
  int width = 0, modes = 0, layers = 0, hidden = 0;  // FNO
  std::vector<float> params;  // deeponet: branch params then trunk params
};

// Parameter counts implied by the architecture (to validate files and C-ABI arrays).
size_t dense_param_count(const std::vector<int32_t>& sizes);
size_t fno_param_count(int width, int modes, int layers, int hidden);

snop_status write_model(const char* path, const ModelFile& m);
snop_status read_model(const char* path, ModelFile& m);

}  // namespace snop_impl
