// Host utilities of the B200 VQMC library (no GPU needed): RNG streams, MADE
// initialisation, graph / TIM generators and the instance text formats.  These are the
// product's own C++ implementations of the reference's host-side functions
// (cited per function); tests check them against the independent oracle.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "vqmc_b200.h"

namespace vqmc_b200 {
void set_error(const std::string& msg);
int status_of(const std::exception& ex);
}  // namespace vqmc_b200

using vqmc_b200::set_error;

namespace {

uint64_t mix_seed(uint64_t seed, uint64_t stream) {  // proj/include/vqmc/common.hpp:56-61
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
std::mt19937_64 make_stream(uint64_t seed, uint64_t stream) {  // common.hpp:64-66
  return std::mt19937_64(mix_seed(seed, stream));
}

using Edges = std::vector<std::pair<int, int>>;

int emit(const Edges& g, int32_t* out, int64_t cap, int64_t* ne) {
  *ne = (int64_t)g.size();
  if (out) {
    if (cap < (int64_t)g.size()) throw std::invalid_argument("edge buffer too small");
    for (size_t t = 0; t < g.size(); ++t) {
      out[2 * t] = g[t].first;
      out[2 * t + 1] = g[t].second;
    }
  }
  return VQMC_OK;
}

// Instance files: '#' comments, whitespace tokens (hamiltonian.cpp:197-216).
std::vector<std::vector<std::string>> read_lines(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::vector<std::vector<std::string>> lines;
  std::string line;
  while (std::getline(in, line)) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    std::istringstream ss(line);
    std::vector<std::string> tok;
    std::string t;
    while (ss >> t) tok.push_back(t);
    if (!tok.empty()) lines.push_back(std::move(tok));
  }
  if (lines.empty()) throw std::runtime_error(path + ": empty instance file");
  return lines;
}

}  // namespace

#define HOST_TRY try {
#define HOST_CATCH                           \
  }                                          \
  catch (const std::exception& ex) {         \
    set_error(ex.what());                    \
    return vqmc_b200::status_of(ex);         \
  }                                          \
  return VQMC_OK;

extern "C" {

uint64_t vqmc_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

int vqmc_default_made_hidden(int n) {  // proj/src/models.cpp:79-82
  const double logn = std::log(static_cast<double>(n));
  return static_cast<int>(std::lround(5.0 * logn * logn));
}

int vqmc_made_init(int n, int h, uint64_t seed, int32_t* degrees_out, double* theta_out) {
  HOST_TRY  // proj/src/models.cpp:84-104
  if (n < 2) throw std::invalid_argument("made_init requires n >= 2");
  if (h < 1) throw std::invalid_argument("made_init requires h >= 1");
  for (int k = 0; k < h; ++k) degrees_out[k] = 1 + (k % (n - 1));
  auto rng = make_stream(seed, 0);
  // uniform_matrix fills row-major (models.cpp:34-42): W1 (h x n) then W2 (n x h)
  std::uniform_real_distribution<double> d1(-1.0 / std::sqrt((double)n), 1.0 / std::sqrt((double)n));
  double* p = theta_out;
  for (int64_t t = 0; t < (int64_t)h * n; ++t) *p++ = d1(rng);
  for (int k = 0; k < h; ++k) *p++ = 0.0;
  std::uniform_real_distribution<double> d2(-1.0 / std::sqrt((double)h), 1.0 / std::sqrt((double)h));
  for (int64_t t = 0; t < (int64_t)n * h; ++t) *p++ = d2(rng);
  for (int i = 0; i < n; ++i) *p++ = 0.0;
  HOST_CATCH
}

int vqmc_stream_uniforms(uint64_t seed, uint64_t stream, uint64_t skip, int64_t count, double* out) {
  HOST_TRY
  auto rng = make_stream(seed, stream);
  std::uniform_real_distribution<double> unit(0.0, 1.0);  // sampler.cpp:39
  for (uint64_t s = 0; s < skip; ++s) (void)unit(rng);
  for (int64_t t = 0; t < count; ++t) out[t] = unit(rng);
  HOST_CATCH
}

int vqmc_random_maxcut_graph(int n, uint64_t seed, int32_t* edges_out, int64_t cap, int64_t* ne) {
  HOST_TRY  // proj/src/hamiltonian.cpp:144-160
  if (n < 1) throw std::invalid_argument("random_maxcut_graph requires n >= 1");
  auto rng = make_stream(seed, 0);
  std::bernoulli_distribution coin(0.5);
  std::vector<uint8_t> b((size_t)n * n);
  for (auto& v : b) v = coin(rng) ? 1 : 0;
  Edges g;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (b[(size_t)i * n + j] || b[(size_t)j * n + i]) g.emplace_back(i, j);
  emit(g, edges_out, cap, ne);
  HOST_CATCH
}

// Random d-regular graph (not in the reference; BASELINE.json configs use it):
// configuration model with rejection, make_stream(seed, 0), index draws r % i.
int vqmc_random_regular_graph(int n, int d, uint64_t seed, int32_t* edges_out, int64_t cap,
                              int64_t* ne) {
  HOST_TRY
  if (n < 1 || d < 0 || d >= n || ((int64_t)n * d) % 2 != 0)
    throw std::invalid_argument("random_regular_graph requires 0 <= d < n and n*d even");
  auto rng = make_stream(seed, 0);
  std::vector<int> pts((size_t)n * d);
  for (int attempt = 0; attempt < 100000; ++attempt) {
    for (int v = 0; v < n; ++v)
      for (int c = 0; c < d; ++c) pts[(size_t)v * d + c] = v;
    for (size_t i = pts.size(); i > 1; --i) std::swap(pts[i - 1], pts[rng() % i]);
    std::set<std::pair<int, int>> seen;
    bool ok = true;
    for (size_t t = 0; t < pts.size(); t += 2) {
      int a = pts[t], c = pts[t + 1];
      if (a == c) { ok = false; break; }
      if (a > c) std::swap(a, c);
      if (!seen.insert({a, c}).second) { ok = false; break; }
    }
    if (!ok) continue;
    Edges g(seen.begin(), seen.end());
    emit(g, edges_out, cap, ne);
    return VQMC_OK;
  }
  throw std::runtime_error("random_regular_graph: too many rejections");
  HOST_CATCH
}

int vqmc_erdos_renyi_graph(int n, double p, uint64_t seed, int32_t* edges_out, int64_t cap,
                           int64_t* ne) {
  HOST_TRY
  if (n < 1 || !(p >= 0.0 && p <= 1.0)) throw std::invalid_argument("erdos_renyi_graph: bad n or p");
  auto rng = make_stream(seed, 0);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  Edges g;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (unit(rng) < p) g.emplace_back(i, j);
  emit(g, edges_out, cap, ne);
  HOST_CATCH
}

// load_graph (hamiltonian.cpp:243-266): "graph <n>" then "edge i j" (1-based).
int vqmc_load_graph(const char* path, int* n_out, int32_t* edges_out, int64_t cap, int64_t* ne) {
  HOST_TRY
  const auto lines = read_lines(path);
  const auto& header = lines.front();
  const std::string p(path);
  if (header.size() != 2 || header[0] != "graph")
    throw std::runtime_error(p + ": expected 'graph <n>' header");
  const int n = std::stoi(header[1]);
  if (n < 1) throw std::runtime_error(p + ": n must be >= 1");
  auto parse = [&](const std::string& t) {
    const int idx = std::stoi(t);
    if (idx < 1 || idx > n) throw std::runtime_error(p + ": index out of range: " + t);
    return idx - 1;
  };
  std::set<std::pair<int, int>> seen;
  Edges g;
  for (size_t k = 1; k < lines.size(); ++k) {
    const auto& t = lines[k];
    if (t[0] != "edge" || t.size() != 3)
      throw std::runtime_error(p + ": malformed line starting with '" + t[0] + "'");
    int i = parse(t[1]), j = parse(t[2]);
    if (i == j) throw std::runtime_error(p + ": self loops are not allowed");
    if (i > j) std::swap(i, j);
    if (!seen.insert({i, j}).second) throw std::runtime_error(p + ": duplicate edge");
    g.emplace_back(i, j);
  }
  *n_out = n;
  emit(g, edges_out, cap, ne);
  HOST_CATCH
}

int vqmc_save_graph(const char* path, int n, const int32_t* edges, int64_t ne) {
  HOST_TRY  // hamiltonian.cpp:236-241
  std::ofstream out(path);
  if (!out) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
  out << "graph " << n << "\n";
  for (int64_t t = 0; t < ne; ++t) out << "edge " << (edges[2 * t] + 1) << " " << (edges[2 * t + 1] + 1) << "\n";
  HOST_CATCH
}

// random_tim (hamiltonian.cpp:126-142): alpha_i ~ U[0,1) for every site, then beta_i ~ U[-1,1),
// then the n(n-1)/2 pairs (row-major i < j) ~ U[-1,1), all from make_stream(seed).
int vqmc_random_tim(int n, uint64_t seed, double* alpha, double* beta, int32_t* pair_i, int32_t* pair_j,
                    double* pair_value) {
  HOST_TRY
  if (n < 1) throw std::invalid_argument("random_tim requires n >= 1");
  auto rng = make_stream(seed, 0);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::uniform_real_distribution<double> symmetric(-1.0, 1.0);
  for (int i = 0; i < n; ++i) alpha[i] = unit(rng);
  for (int i = 0; i < n; ++i) beta[i] = symmetric(rng);
  int64_t t = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j, ++t) {
      pair_i[t] = i;
      pair_j[t] = j;
      pair_value[t] = symmetric(rng);
    }
  HOST_CATCH
}

// load_spec (hamiltonian.cpp:204-234): "tim <n>", then "alpha i v" / "beta i v" / "pair i j v"
// (1-based; i < j).  Call with alpha == NULL to get *n_out and *num_pairs first.  Validation
// (negative alpha, duplicate pairs) is HamiltonianSpec::validate's, done by vqmc_gpu_set_spec.
int vqmc_load_spec(const char* path, int* n_out, double* alpha, double* beta, int32_t* pair_i, int32_t* pair_j,
                   double* pair_value, int64_t cap, int64_t* num_pairs) {
  HOST_TRY
  const auto lines = read_lines(path);
  const auto& header = lines.front();
  const std::string p(path);
  if (header.size() != 2 || header[0] != "tim") throw std::runtime_error(p + ": expected 'tim <n>' header");
  const int n = std::stoi(header[1]);
  if (n < 1) throw std::runtime_error(p + ": n must be >= 1");
  auto parse = [&](const std::string& t) {
    const int idx = std::stoi(t);
    if (idx < 1 || idx > n) throw std::runtime_error(p + ": index out of range: " + t);
    return idx - 1;
  };
  std::vector<double> a(n, 0.0), b(n, 0.0);
  std::vector<int32_t> pi, pj;
  std::vector<double> pv;
  for (size_t k = 1; k < lines.size(); ++k) {
    const auto& t = lines[k];
    if (t[0] == "alpha" && t.size() == 3) {
      a[parse(t[1])] = std::stod(t[2]);
    } else if (t[0] == "beta" && t.size() == 3) {
      b[parse(t[1])] = std::stod(t[2]);
    } else if (t[0] == "pair" && t.size() == 4) {
      const int i = parse(t[1]), j = parse(t[2]);
      if (i >= j) throw std::runtime_error(p + ": pair indices must satisfy i < j");
      pi.push_back(i);
      pj.push_back(j);
      pv.push_back(std::stod(t[3]));
    } else {
      throw std::runtime_error(p + ": malformed line starting with '" + t[0] + "'");
    }
  }
  *n_out = n;
  *num_pairs = (int64_t)pi.size();
  if (alpha) {
    if (cap < (int64_t)pi.size()) throw std::invalid_argument("pair buffer too small");
    std::memcpy(alpha, a.data(), sizeof(double) * n);
    std::memcpy(beta, b.data(), sizeof(double) * n);
    for (size_t t = 0; t < pi.size(); ++t) {
      pair_i[t] = pi[t];
      pair_j[t] = pj[t];
      pair_value[t] = pv[t];
    }
  }
  HOST_CATCH
}

// save_spec (hamiltonian.cpp:162-177): zero fields are omitted, 17 significant digits.
int vqmc_save_spec(const char* path, int n, const double* alpha, const double* beta, const int32_t* pair_i,
                   const int32_t* pair_j, const double* pair_value, int64_t num_pairs) {
  HOST_TRY
  std::ofstream out(path);
  if (!out) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
  out.precision(17);
  out << "tim " << n << "\n";
  for (int i = 0; i < n; ++i)
    if (alpha[i] != 0.0) out << "alpha " << (i + 1) << " " << alpha[i] << "\n";
  for (int i = 0; i < n; ++i)
    if (beta[i] != 0.0) out << "beta " << (i + 1) << " " << beta[i] << "\n";
  for (int64_t t = 0; t < num_pairs; ++t)
    out << "pair " << (pair_i[t] + 1) << " " << (pair_j[t] + 1) << " " << pair_value[t] << "\n";
  HOST_CATCH
}

}  // extern "C"
