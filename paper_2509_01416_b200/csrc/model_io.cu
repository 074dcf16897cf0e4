// model_io.cu — host-side model-file writer/reader (format: model_io.h) and the C-ABI entry
// points that need no device: snop_model_write_deeponet / snop_model_write_fno /
// snop_model_inspect. snop_op_save / snop_op_load (op_capi.cu) build on these.
//
// The file is assembled in memory and written with one fwrite; the reader slurps the file and
// parses it with a bounds-checked cursor, so a truncated file can never be read past its end.
// Integers and doubles are little-endian regardless of host order (byte-wise encode), the digest
// is FNV-1a-64 (offset 0xcbf29ce484222325, prime 0x100000001b3) over every record byte
// (binary_io.cpp:12-17), appended as a little-endian u64 (binary_io.cpp:73-83).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "model_io.h"

namespace snop_impl {

void set_error(const std::string& msg);

namespace {

constexpr const char* kMagic = "SNOP-MODEL";
constexpr uint32_t kVersion = 1;
constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull, kFnvPrime = 0x100000001b3ull;

uint64_t fnv1a(const uint8_t* p, size_t n, uint64_t h = kFnvOffset) {
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * kFnvPrime;
  return h;
}

class Out {
 public:
  void le(uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) buf.push_back(static_cast<uint8_t>(v >> (8 * i)));
  }
  void u8(uint8_t v) { buf.push_back(v); }
  void u32(uint32_t v) { le(v, 4); }
  void u64(uint64_t v) { le(v, 8); }
  void f64(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    le(u, 8);
  }
  void str(const std::string& s) {
    u32(static_cast<uint32_t>(s.size()));
    buf.insert(buf.end(), s.begin(), s.end());
  }
  std::vector<uint8_t> buf;
};

struct Truncated {};

class In {
 public:
  In(const uint8_t* p, size_t n) : p_(p), n_(n) {}
  uint64_t le(int bytes) {
    need(bytes);
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(p_[pos + i]) << (8 * i);
    pos += bytes;
    return v;
  }
  uint8_t u8() { return static_cast<uint8_t>(le(1)); }
  uint32_t u32() { return static_cast<uint32_t>(le(4)); }
  uint64_t u64() { return le(8); }
  double f64() {
    const uint64_t u = le(8);
    double v;
    std::memcpy(&v, &u, 8);
    return v;
  }
  std::string str(size_t max_len) {
    const uint32_t n = u32();
    if (n > max_len) throw Truncated{};
    need(n);
    std::string s(reinterpret_cast<const char*>(p_ + pos), n);
    pos += n;
    return s;
  }
  size_t pos = 0;

 private:
  void need(size_t k) {
    if (k > n_ - pos) throw Truncated{};
  }
  const uint8_t* p_;
  size_t n_;
};

snop_status io_error(const std::string& m) {
  set_error(m);
  return SNOP_IO_ERROR;
}
snop_status bad(const std::string& m) {
  set_error(m);
  return SNOP_INVALID_ARGUMENT;
}

snop_status validate(const ModelFile& m) {
  if (!(m.grid.length_cm > 0.0) || m.grid.n_cells < 1) return bad("model: bad grid");
  if (m.act < 0 || m.act > 2) return bad("model: activation must be relu(0), tanh(1) or gelu(2)");
  size_t want = 0;
  if (m.arch == SNOP_ARCH_DEEPONET) {
    if (m.bs.size() < 2 || m.ts.size() < 2) return bad("model: networks need >= 2 layer sizes");
    for (int32_t s : m.bs) if (s < 1) return bad("model: bad branch size");
    for (int32_t s : m.ts) if (s < 1) return bad("model: bad trunk size");
    if (m.bs.back() != m.ts.back()) return bad("model: branch/trunk output widths differ");
    want = dense_param_count(m.bs) + dense_param_count(m.ts);
  } else if (m.arch == SNOP_ARCH_FNO) {
    if (m.width < 1 || m.modes < 1 || m.layers < 0 || m.hidden < 1) return bad("model: bad FNO architecture");
    want = fno_param_count(m.width, m.modes, m.layers, m.hidden);
  } else {
    return bad("model: unknown architecture");
  }
  if (m.params.size() != want) return bad("model: parameter count does not match the architecture");
  return SNOP_OK;
}

}  // namespace

size_t dense_param_count(const std::vector<int32_t>& s) {
  size_t n = 0;
  for (size_t l = 0; l + 1 < s.size(); ++l) n += (size_t)s[l] * s[l + 1] + s[l + 1];
  return n;
}

size_t fno_param_count(int C, int M, int L, int H) {
  const size_t c = C, m = M;
  return 3 * c + (size_t)L * (2 * m * c * c + c * c + c) + (size_t)H * c + 2 * (size_t)H + 1;
}

snop_status write_model(const char* path, const ModelFile& m) {
  if (!path) return bad("path is NULL");
  const snop_status v = validate(m);
  if (v != SNOP_OK) return v;
  Out o;
  o.str(kMagic);
  o.u32(kVersion);
  o.str(m.arch == SNOP_ARCH_DEEPONET ? "deeponet" : "fno");
  o.f64(m.grid.length_cm);
  o.u64((uint64_t)m.grid.n_cells);
  o.f64(m.tstar);
  o.f64(m.sstar);
  o.u32((uint32_t)m.act);
  if (m.arch == SNOP_ARCH_DEEPONET) {
    o.u32((uint32_t)m.bs.size());
    for (int32_t s : m.bs) o.u64((uint64_t)s);
    o.u32((uint32_t)m.ts.size());
    for (int32_t s : m.ts) o.u64((uint64_t)s);
    o.u8(m.has_bias0 ? 1 : 0);
    o.f64(m.has_bias0 ? (double)m.bias0 : 0.0);
  } else {
    o.u64((uint64_t)m.width);
    o.u64((uint64_t)m.modes);
    o.u64((uint64_t)m.layers);
    o.u64((uint64_t)m.hidden);
  }
  o.u64(m.params.size());
  for (float x : m.params) o.f64((double)x);
  const uint64_t digest = fnv1a(o.buf.data(), o.buf.size());
  o.u64(digest);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_error(std::string("cannot open for writing: ") + path);
  const bool ok = std::fwrite(o.buf.data(), 1, o.buf.size(), f) == o.buf.size();
  const bool closed = std::fclose(f) == 0;
  if (!ok || !closed) return io_error(std::string("short write: ") + path);
  return SNOP_OK;
}

snop_status read_model(const char* path, ModelFile& m) {
  if (!path) return bad("path is NULL");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return io_error(std::string("cannot open for reading: ") + path);
  std::vector<uint8_t> buf;
  uint8_t chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
  const bool err = std::ferror(f) != 0;
  std::fclose(f);
  if (err) return io_error(std::string("read failed: ") + path);
  if (buf.size() < 8) return io_error("checksum missing (truncated file)");
  const size_t body = buf.size() - 8;
  try {
    In in(buf.data(), body);
    if (in.str(64) != kMagic) return io_error("not a snop model file (bad magic)");
    const uint32_t version = in.u32();
    if (version != kVersion)
      return io_error("model file version " + std::to_string(version) + " unsupported (expected 1)");
    const std::string arch = in.str(64);
    if (arch == "deeponet") m.arch = SNOP_ARCH_DEEPONET;
    else if (arch == "fno") m.arch = SNOP_ARCH_FNO;
    else return io_error("unknown architecture tag '" + arch + "'");
    m.grid.length_cm = in.f64();
    const uint64_t nc = in.u64();
    if (nc < 1 || nc > (1u << 30)) return io_error("implausible n_cells (corrupt file?)");
    m.grid.n_cells = (int32_t)nc;
    m.grid.reserved = 0;
    m.tstar = in.f64();
    m.sstar = in.f64();
    m.act = (int)in.u32();
    auto sizes = [&](std::vector<int32_t>& v) {
      const uint32_t n = in.u32();
      if (n > 64) throw Truncated{};
      v.resize(n);
      for (auto& s : v) {
        const uint64_t x = in.u64();
        if (x > (1u << 24)) throw Truncated{};
        s = (int32_t)x;
      }
    };
    if (m.arch == SNOP_ARCH_DEEPONET) {
      sizes(m.bs);
      sizes(m.ts);
      m.has_bias0 = in.u8() != 0;
      m.bias0 = (float)in.f64();
    } else {
      uint64_t a[4];
      for (auto& x : a) {
        x = in.u64();
        if (x > (1u << 20)) throw Truncated{};
      }
      m.width = (int)a[0];
      m.modes = (int)a[1];
      m.layers = (int)a[2];
      m.hidden = (int)a[3];
    }
    const uint64_t np = in.u64();
    if (np > (body - in.pos) / 8) throw Truncated{};
    m.params.resize(np);
    for (auto& x : m.params) x = (float)in.f64();
    if (in.pos != body) return io_error("checksum mismatch (corrupt file: trailing bytes)");
  } catch (const Truncated&) {
    return io_error("unexpected end of file (truncated or corrupt model file)");
  }
  uint64_t stored = 0;
  for (int i = 0; i < 8; ++i) stored |= static_cast<uint64_t>(buf[body + i]) << (8 * i);
  if (stored != fnv1a(buf.data(), body)) return io_error("checksum mismatch (corrupt file)");
  const snop_status v = validate(m);
  if (v != SNOP_OK) return io_error("inconsistent model record (corrupt file?)");
  return SNOP_OK;
}

}  // namespace snop_impl

using namespace snop_impl;

extern "C" {

snop_status snop_model_write_deeponet(const char* path, const snop_grid* grid, double tstar, double sstar,
                                      int32_t act, int32_t nb, const int32_t* bs, const float* bp, int32_t nt,
                                      const int32_t* ts, const float* tp, int32_t has_bias0, float bias0) {
  if (!grid || !bs || !bp || !ts || !tp || nb < 2 || nt < 2) return bad("NULL argument or too few layers");
  ModelFile m;
  m.arch = SNOP_ARCH_DEEPONET;
  m.grid = *grid;
  m.tstar = tstar;
  m.sstar = sstar;
  m.act = act;
  m.bs.assign(bs, bs + nb);
  m.ts.assign(ts, ts + nt);
  for (int32_t s : m.bs) if (s < 1) return bad("bad branch size");
  for (int32_t s : m.ts) if (s < 1) return bad("bad trunk size");
  const size_t nbp = dense_param_count(m.bs), ntp = dense_param_count(m.ts);
  m.params.assign(bp, bp + nbp);
  m.params.insert(m.params.end(), tp, tp + ntp);
  m.has_bias0 = has_bias0 != 0;
  m.bias0 = bias0;
  return write_model(path, m);
}

snop_status snop_model_write_fno(const char* path, const snop_grid* grid, double tstar, double sstar, int32_t act,
                                 int32_t width, int32_t modes, int32_t layers, int32_t hidden, const float* params) {
  if (!grid || !params) return bad("NULL argument");
  if (width < 1 || modes < 1 || layers < 0 || hidden < 1) return bad("bad FNO architecture");
  ModelFile m;
  m.arch = SNOP_ARCH_FNO;
  m.grid = *grid;
  m.tstar = tstar;
  m.sstar = sstar;
  m.act = act;
  m.width = width;
  m.modes = modes;
  m.layers = layers;
  m.hidden = hidden;
  m.params.assign(params, params + fno_param_count(width, modes, layers, hidden));
  return write_model(path, m);
}

snop_status snop_model_inspect(const char* path, snop_model_info* info) {
  if (!info) return bad("info is NULL");
  ModelFile m;
  const snop_status s = read_model(path, m);
  if (s != SNOP_OK) return s;
  std::memset(info, 0, sizeof *info);
  info->arch = m.arch;
  info->grid = m.grid;
  info->sigma_t_star = m.tstar;
  info->sigma_s0_star = m.sstar;
  info->activation = m.act;
  info->n_params = (int64_t)m.params.size();
  if (m.arch == SNOP_ARCH_DEEPONET) {
    info->n_branch = (int32_t)m.bs.size();
    info->n_trunk = (int32_t)m.ts.size();
    info->latent = m.bs.back();
    info->has_bias0 = m.has_bias0 ? 1 : 0;
    info->bias0 = m.bias0;
  } else {
    info->width = m.width;
    info->modes = m.modes;
    info->layers = m.layers;
    info->hidden = m.hidden;
  }
  return SNOP_OK;
}

// Dataset record (format version 1), same container as the model file:
//   string "SNOP-DATASET", u32 version, u64 n_samples, u64 n_cells, f64 length_cm, u32 order,
//   f64 mean, f64 variance, f64 length_scale, f64 jitter, u64 seed, f64 sigma_t*, f64 sigma_s0*,
//   f64 tolerance, f64 sources[n_samples*n_cells], f64 fluxes[n_samples*n_cells], u64 digest.
snop_status snop_dataset_write(const char* path, const snop_dataset_info* info, const double* sources,
                               const double* fluxes) {
  if (!path || !info || !sources || !fluxes) return bad("NULL argument");
  if (info->n_samples < 0 || info->grid.n_cells < 1 || !(info->grid.length_cm > 0.0)) return bad("bad dataset header");
  const size_t N = (size_t)info->n_samples * info->grid.n_cells;
  Out o;
  o.buf.reserve(128 + 16 * N);
  o.str("SNOP-DATASET");
  o.u32(1);
  o.u64((uint64_t)info->n_samples);
  o.u64((uint64_t)info->grid.n_cells);
  o.f64(info->grid.length_cm);
  o.u32((uint32_t)info->order);
  o.f64(info->spec.mean);
  o.f64(info->spec.variance);
  o.f64(info->spec.length_scale_cm);
  o.f64(info->spec.jitter);
  o.u64(info->spec.seed);
  o.f64(info->sigma_t_star);
  o.f64(info->sigma_s0_star);
  o.f64(info->tolerance);
  for (size_t i = 0; i < N; ++i) o.f64(sources[i]);
  for (size_t i = 0; i < N; ++i) o.f64(fluxes[i]);
  o.u64(fnv1a(o.buf.data(), o.buf.size()));
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_error(std::string("cannot open for writing: ") + path);
  const bool ok = std::fwrite(o.buf.data(), 1, o.buf.size(), f) == o.buf.size();
  if (std::fclose(f) != 0 || !ok) return io_error(std::string("short write: ") + path);
  // human-readable manifest alongside
  const std::string mpath = std::string(path) + ".txt";
  std::FILE* m = std::fopen(mpath.c_str(), "w");
  if (!m) return io_error("cannot open manifest for writing: " + mpath);
  std::fprintf(m,
               "format = SNOP-DATASET v1\nn_samples = %lld\nn_cells = %d\nlength_cm = %.17g\nquadrature_order = %d\n"
               "grf_mean = %.17g\ngrf_variance = %.17g\ngrf_length_scale_cm = %.17g\ngrf_jitter = %.17g\n"
               "grf_seed = %llu\nsigma_t_star = %.17g\nsigma_s0_star = %.17g\nsolver_tolerance = %.17g\n"
               "layout = sources[n_samples][n_cells] then fluxes[n_samples][n_cells], f64 little-endian\n"
               "digest_fnv1a64 = %016llx\n",
               (long long)info->n_samples, info->grid.n_cells, info->grid.length_cm, info->order, info->spec.mean,
               info->spec.variance, info->spec.length_scale_cm, info->spec.jitter,
               (unsigned long long)info->spec.seed, info->sigma_t_star, info->sigma_s0_star, info->tolerance,
               (unsigned long long)fnv1a(o.buf.data(), o.buf.size() - 8));
  if (std::fclose(m) != 0) return io_error("manifest write failed: " + mpath);
  return SNOP_OK;
}

snop_status snop_dataset_read(const char* path, snop_dataset_info* info, double* sources, double* fluxes) {
  if (!path || !info) return bad("NULL argument");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return io_error(std::string("cannot open for reading: ") + path);
  std::vector<uint8_t> buf;
  uint8_t chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
  std::fclose(f);
  if (buf.size() < 8) return io_error("checksum missing (truncated file)");
  const size_t body = buf.size() - 8;
  snop_dataset_info h{};
  size_t data_pos = 0;
  try {
    In in(buf.data(), body);
    if (in.str(64) != "SNOP-DATASET") return io_error("not a snop dataset file (bad magic)");
    const uint32_t version = in.u32();
    if (version != 1) return io_error("dataset file version " + std::to_string(version) + " unsupported (expected 1)");
    h.n_samples = (int64_t)in.u64();
    const uint64_t nc = in.u64();
    if (nc < 1 || nc > (1u << 30) || h.n_samples < 0) throw Truncated{};
    h.grid.n_cells = (int32_t)nc;
    h.grid.length_cm = in.f64();
    h.order = (int32_t)in.u32();
    h.spec.mean = in.f64();
    h.spec.variance = in.f64();
    h.spec.length_scale_cm = in.f64();
    h.spec.jitter = in.f64();
    h.spec.seed = in.u64();
    h.sigma_t_star = in.f64();
    h.sigma_s0_star = in.f64();
    h.tolerance = in.f64();
    data_pos = in.pos;
    const size_t N = (size_t)h.n_samples * nc;
    if (N > (body - data_pos) / 16 || data_pos + 16 * N != body) throw Truncated{};
  } catch (const Truncated&) {
    return io_error("unexpected end of file (truncated or corrupt dataset file)");
  }
  uint64_t stored = 0;
  for (int i = 0; i < 8; ++i) stored |= static_cast<uint64_t>(buf[body + i]) << (8 * i);
  if (stored != fnv1a(buf.data(), body)) return io_error("checksum mismatch (corrupt file)");
  *info = h;
  const size_t N = (size_t)h.n_samples * h.grid.n_cells;
  In data(buf.data() + data_pos, 16 * N);
  for (size_t i = 0; i < N; ++i) {
    const double v = data.f64();
    if (sources) sources[i] = v;
  }
  for (size_t i = 0; i < N; ++i) {
    const double v = data.f64();
    if (fluxes) fluxes[i] = v;
  }
  return SNOP_OK;
}

}  // extern "C"
