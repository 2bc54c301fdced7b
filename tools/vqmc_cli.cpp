// vqmc — command-line drop-in for the reference's `vqmc` tool (proj/tools/vqmc.cpp) on the
// B200 path.  Same subcommands, flags, config-file precedence, output files and exit codes
// (0 ok, 1 usage, 2 numerical, 3 sample-test reject; vqmc.cpp:35-37) for the north-star
// workload (Max-Cut, MADE, AUTO sampler, ADAM or SGD + SR) and TIM instances (ADAM).
// Configurations outside that path (RBM/MCMC, plain SGD, the TIM ground-state eigensolver) are
// rejected as usage errors with an explicit message.  `--gpus G` spreads the `--workers` over G
// GPUs (one host thread and NCCL rank each).
//
// CLI11 and nlohmann/json are not available in this image; the parser below implements the
// subset of CLI11 behaviour the reference relies on: `--flag value` and `--flag=value`,
// repeated options take the last value (TakeLast), and `--config` key=value entries are
// spliced in before the explicit flags so the command line wins (vqmc.cpp:42-73, 490-504).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "vqmc_b200/vqmc.hpp"

namespace {

constexpr int kExitUsage = 1;
constexpr int kExitNumerical = 2;
constexpr int kExitRejected = 3;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------------------
// Arguments
// ---------------------------------------------------------------------------------------
struct Args {
  std::map<std::string, std::string> opt;  // last value wins
  std::set<std::string> flags;
  bool has(const std::string& k) const { return opt.count(k) > 0; }
  std::string get(const std::string& k, const std::string& d) const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
  long long geti(const std::string& k, long long d) const {
    if (!has(k)) return d;
    try {
      size_t pos = 0;
      const long long v = std::stoll(opt.at(k), &pos);
      if (pos != opt.at(k).size()) throw std::invalid_argument("");
      return v;
    } catch (...) {
      throw UsageError("--" + k + ": not an integer: " + opt.at(k));
    }
  }
  double getd(const std::string& k, double d) const {
    if (!has(k)) return d;
    try {
      size_t pos = 0;
      const double v = std::stod(opt.at(k), &pos);
      if (pos != opt.at(k).size()) throw std::invalid_argument("");
      return v;
    } catch (...) {
      throw UsageError("--" + k + ": not a number: " + opt.at(k));
    }
  }
};

Args parse(const std::vector<std::string>& argv, const std::set<std::string>& options,
           const std::set<std::string>& flag_names) {
  Args a;
  for (size_t i = 0; i < argv.size(); ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + s);
    s = s.substr(2);
    std::string val;
    bool has_val = false;
    const auto eq = s.find('=');
    if (eq != std::string::npos) {
      val = s.substr(eq + 1);
      s = s.substr(0, eq);
      has_val = true;
    }
    if (flag_names.count(s)) {
      a.flags.insert(s);
      continue;
    }
    if (!options.count(s)) throw UsageError("The following argument was not expected: --" + s);
    if (!has_val) {
      if (i + 1 >= argv.size()) throw UsageError("--" + s + " requires a value");
      val = argv[++i];
    }
    a.opt[s] = val;
  }
  return a;
}

// vqmc.cpp:42-73: flat key=value files, booleans only for the three flag keys.
std::vector<std::string> config_file_args(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw UsageError("cannot open config file: " + path);
  std::vector<std::string> args;
  std::string line;
  auto trim = [](std::string s) {
    const auto f = s.find_first_not_of(" \t\r");
    if (f == std::string::npos) return std::string();
    return s.substr(f, s.find_last_not_of(" \t\r") - f + 1);
  };
  while (std::getline(in, line)) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    const auto eq = line.find('=');
    if (eq == std::string::npos) {
      if (line.find_first_not_of(" \t\r") != std::string::npos)
        throw UsageError("config line is not key=value: " + line);
      continue;
    }
    const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
    if (key.empty()) throw UsageError("config line is not key=value: " + line);
    if (key == "mcmc-reburn" || key == "sr-fallback" || key == "sr-uncentered") {
      if (value == "true" || value == "1" || value == "yes") args.push_back("--" + key);
      continue;
    }
    args.push_back("--" + key);
    args.push_back(value);
  }
  return args;
}

std::string sniff_header(const std::string& path) {  // vqmc.cpp:76-89
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open instance file: " + path);
  std::string line;
  while (std::getline(in, line)) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    std::istringstream ss(line);
    std::string tok;
    if (ss >> tok) return tok;
  }
  throw std::runtime_error("empty instance file: " + path);
}

// shortest round-trip formatting of a double (as nlohmann::json prints numbers)
std::string jnum(double v) {
  if (std::isnan(v) || std::isinf(v)) return "null";
  if (v == std::floor(v) && std::fabs(v) < 1e15) {
    char b[64];
    std::snprintf(b, sizeof b, "%.1f", v);
    return b;
  }
  for (int p = 1; p <= 17; ++p) {
    char b[64];
    std::snprintf(b, sizeof b, "%.*g", p, v);
    if (std::strtod(b, nullptr) == v) return b;
  }
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

// A tiny ordered JSON object printer with nlohmann's dump(2) layout (keys sorted).
struct JObj {
  std::map<std::string, std::string> kv;  // values already serialised
  std::string dump(int indent = 2, int level = 1) const {
    std::string pad((size_t)indent * level, ' '), pad0((size_t)indent * (level - 1), ' ');
    std::string o = "{\n";
    size_t i = 0;
    for (const auto& [k, v] : kv) {
      o += pad + jstr(k) + ": " + v;
      o += (++i < kv.size()) ? ",\n" : "\n";
    }
    return o + pad0 + "}";
  }
};

// ---------------------------------------------------------------------------------------
// solve (vqmc.cpp:194-263)
// ---------------------------------------------------------------------------------------
int run_solve(const Args& a) {
  const std::string problem = a.get("problem", "tim");
  const std::string model = a.get("model", "made");
  const std::string optimizer = a.get("optimizer", "adam");
  if (problem != "tim" && problem != "maxcut") throw UsageError("--problem: not in {tim, maxcut}");
  if (model != "made" && model != "rbm") throw UsageError("--model: not in {made, rbm}");
  if (optimizer != "sgd" && optimizer != "adam" && optimizer != "sgd_sr")
    throw UsageError("--optimizer: not in {sgd, adam, sgd_sr}");
  if (a.has("sampler")) {  // vqmc.cpp:516-523
    const std::string expected = model == "made" ? "auto" : "mcmc";
    if (a.get("sampler", "") != expected)
      throw UsageError("--sampler " + a.get("sampler", "") + " cannot be used with --model " + model +
                       " (made pairs with auto, rbm with mcmc)");
  }
  if (model != "made") throw UsageError("the B200 path implements MADE + AUTO (RBM/MCMC is out of scope)");
  if (optimizer == "sgd") throw UsageError("the B200 path implements ADAM and SGD + SR (plain sgd is out of scope)");

  vqmc::RunConfig cfg;
  cfg.seed = (uint64_t)a.geti("seed", 0);
  cfg.hidden = (int)a.geti("hidden", 0);
  cfg.lr = a.getd("lr", 0.0);
  cfg.iterations = (int)a.geti("iterations", 300);
  cfg.minibatch = (int)a.geti("minibatch", 1024);
  cfg.eval_batch = (int)a.geti("eval-batch", 1024);
  cfg.workers = (int)a.geti("workers", 1);
  cfg.device = (int)a.geti("device", 0);
  cfg.gpus = (int)a.geti("gpus", 1);
  cfg.reference_streams = a.flags.count("reference-streams") > 0;
  if (optimizer == "sgd_sr") {  // vqmc.cpp:416-425
    cfg.optimizer = vqmc::OptimizerKind::kSgdSr;
    cfg.sr.lambda = a.getd("sr-lambda", cfg.sr.lambda);
    cfg.sr.tol = a.getd("sr-tol", cfg.sr.tol);
    cfg.sr.max_iterations = (int)a.geti("sr-maxiter", cfg.sr.max_iterations);
    cfg.sr.fallback = a.flags.count("sr-fallback") > 0;
    cfg.sr.centered = a.flags.count("sr-uncentered") == 0;
  }
  if (a.has("target")) cfg.target = a.getd("target", 0.0);
  const std::string instance = a.get("instance", "");
  const int n = (int)a.geti("n", 0);
  const std::string out_dir = a.get("out", ".");

  // resolve_instance (vqmc.cpp:119-140): a file wins over generation
  vqmc::Graph g;
  try {
    if (!instance.empty()) {
      if (sniff_header(instance) == "graph") {
        g = vqmc::load_graph(instance);
      } else {
        cfg.spec = vqmc::load_spec(instance);
      }
    } else if (n < 1) {
      throw UsageError("--n: either --instance or --n is required");
    } else if (problem == "maxcut") {
      g = vqmc::random_maxcut_graph(n, cfg.seed);
    } else {
      cfg.spec = vqmc::random_tim(n, cfg.seed);
    }
    if (!cfg.spec) cfg.maxcut = vqmc::maxcut_spec(g);
  } catch (const UsageError&) {
    throw;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
  const bool is_maxcut = cfg.maxcut.has_value();
  if (!is_maxcut) {
    g.n = cfg.spec->n;
    if (cfg.optimizer == vqmc::OptimizerKind::kSgdSr)
      throw UsageError("the B200 path trains TIM instances with ADAM (sgd_sr is implemented for Max-Cut)");
  }

  if (std::getenv("VQMC_CLI_DRYRUN")) {  // test hook: print the resolved configuration
    std::cout << "problem " << (is_maxcut ? "maxcut" : "tim") << " gpus " << cfg.gpus << "\n";
    std::cout << "n " << g.n << " edges " << g.edges.size() << " seed " << cfg.seed << " iterations "
              << cfg.iterations << " minibatch " << cfg.minibatch << " eval_batch " << cfg.eval_batch
              << " workers " << cfg.workers << " hidden " << cfg.hidden << " lr " << cfg.lr << "\n";
    return 0;
  }

  vqmc::RunResult res;
  try {
    res = vqmc::train(cfg);
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return kExitNumerical;
  }

  std::filesystem::create_directories(out_dir);
  {  // write_curve (vqmc.cpp:181-192)
    std::ofstream out(out_dir + "/curve.csv");
    if (!out) throw std::runtime_error("cannot write " + out_dir + "/curve.csv");
    out << "iter,energy_mean,energy_std,grad_norm,time_s\n";
    char row[256];
    for (size_t i = 0; i < res.stats.size(); ++i) {
      std::snprintf(row, sizeof row, "%zu,%.17g,%.17g,%.17g,%.17g\n", i, res.stats[i].energy_mean,
                    res.stats[i].energy_std, res.stats[i].grad_norm, res.stats[i].wall_time);
      out << row;
    }
  }
  JObj c;  // config_echo (vqmc.cpp:142-179)
  c.kv["problem"] = jstr(is_maxcut ? "maxcut" : "tim");
  c.kv["instance"] = jstr(instance);
  c.kv["n"] = std::to_string(g.n);
  c.kv["seed"] = std::to_string(cfg.seed);
  c.kv["model"] = jstr("made");
  c.kv["sampler"] = jstr("auto");
  c.kv["hidden"] = std::to_string(cfg.hidden > 0 ? cfg.hidden : vqmc::default_made_hidden(g.n));
  c.kv["optimizer"] = jstr(optimizer);
  c.kv["lr"] = jnum(vqmc::resolve_lr(cfg));
  c.kv["iterations"] = std::to_string(cfg.iterations);
  c.kv["workers"] = std::to_string(cfg.workers);
  c.kv["minibatch"] = std::to_string(cfg.minibatch);
  c.kv["eval_batch"] = std::to_string(cfg.eval_batch);
  if (cfg.optimizer == vqmc::OptimizerKind::kSgdSr) {  // config_echo (vqmc.cpp:170-176)
    c.kv["sr_lambda"] = jnum(cfg.sr.lambda);
    c.kv["sr_tol"] = jnum(cfg.sr.tol);
    c.kv["sr_maxiter"] = std::to_string(cfg.sr.max_iterations);
    c.kv["sr_fallback"] = cfg.sr.fallback ? "true" : "false";
    c.kv["sr_centered"] = cfg.sr.centered ? "true" : "false";
  }
  if (cfg.target) c.kv["target"] = jnum(*cfg.target);
  JObj ph;
  ph.kv["sample"] = jnum(res.phases.sample);
  ph.kv["estimate"] = jnum(res.phases.estimate);
  ph.kv["reduce"] = jnum(res.phases.reduce);
  ph.kv["update"] = jnum(res.phases.update);
  JObj s;
  s.kv["config"] = c.dump(2, 2);
  s.kv["final_energy"] = jnum(res.final_energy);
  s.kv["final_energy_std"] = jnum(res.final_energy_std);
  s.kv["iterations_run"] = std::to_string(res.stats.size());
  s.kv["total_time_s"] = jnum(res.total_time);
  s.kv["replicas_identical"] = res.replicas_identical ? "true" : "false";
  s.kv["phase_times_s"] = ph.dump(2, 2);
  if (res.best_cut) {
    s.kv["best_cut"] = jnum(*res.best_cut);
    s.kv["mean_cut"] = jnum(*res.mean_cut);
  }
  if (res.hit_time) {
    s.kv["hit_time_s"] = jnum(*res.hit_time);
    s.kv["hit_iteration"] = std::to_string(res.hit_iteration);
  }
  std::ofstream(out_dir + "/summary.json") << s.dump() << "\n";
  if (a.has("save-model")) vqmc::save_model(*res.made, a.get("save-model", ""));
  std::cout << "final energy " << res.final_energy << " +- " << res.final_energy_std << "\n";
  if (res.best_cut) std::cout << "best cut " << *res.best_cut << " mean cut " << *res.mean_cut << "\n";
  std::cout << "wrote " << out_dir << "/curve.csv and " << out_dir << "/summary.json\n";
  return 0;
}

// oracle (vqmc.cpp:291-313): brute-force max cut of a graph instance (oracle.cpp:80-110).
int run_oracle(const Args& a) {
  if (!a.has("instance")) throw UsageError("--instance is required");
  const std::string path = a.get("instance", "");
  vqmc::Graph g;
  try {
    if (sniff_header(path) != "graph") throw UsageError("TIM ground-state oracle is outside the B200 path");
    g = vqmc::load_graph(path);
  } catch (const UsageError&) {
    throw;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
  if (g.n > 24) throw UsageError("brute_force_maxcut is capped at n <= 24");
  long best = -1;
  uint64_t arg = 0;
  for (uint64_t mask = 0; mask < (uint64_t(1) << (g.n - 1)); ++mask) {
    long cut = 0;
    for (const auto& [i, j] : g.edges) cut += ((mask >> (g.n - 1 - i)) & 1u) != ((mask >> (g.n - 1 - j)) & 1u);
    if (cut > best) {
      best = cut;
      arg = mask;
    }
  }
  std::cout << "max cut " << best << "\nassignment";
  for (int i = 0; i < g.n; ++i) std::cout << " " << ((arg >> (g.n - 1 - i)) & 1u);
  std::cout << "\n";
  return 0;
}

// sample-test (vqmc.cpp:315-373) for MADE: GoF of GPU samples against the enumerated
// distribution (the enumeration is exp(log_prob) of every configuration, also on the GPU).
int run_sample_test(const Args& a) {
  const std::string model = a.get("model", "made");
  if (model != "made") throw UsageError("sample-test: RBM/MCMC is outside the B200 path");
  const uint64_t seed = (uint64_t)a.geti("seed", 0);
  const long samples = (long)a.geti("samples", 100000);
  vqmc::MadeModel m;
  if (a.has("checkpoint")) {
    m = vqmc::load_made(a.get("checkpoint", ""));
  } else {
    const int n = (int)a.geti("n", 0);
    if (n < 1) throw UsageError("--n: required without --checkpoint");
    const int h = (int)a.geti("hidden", 0);
    m = vqmc::made_init(n, h > 0 ? h : vqmc::default_made_hidden(n), seed);
  }
  if (m.n > 16) throw UsageError("enumerate_distribution is capped at n <= 16");
  const int n = m.n;
  const uint64_t count = uint64_t(1) << n;
  vqmc::ConfigBatch all((int)count, n);
  for (uint64_t idx = 0; idx < count; ++idx)
    for (int i = 0; i < n; ++i) all((int)idx, i) = (idx >> (n - 1 - i)) & 1u;
  const vqmc::Vector lp = vqmc::log_prob(m, all);
  auto rng = vqmc::make_stream(seed, 17);
  const vqmc::SampleBatch batch = vqmc::auto_sample(m, (int)samples, rng);
  std::vector<long> counts(count, 0);
  for (int b = 0; b < batch.configs.rows(); ++b) {
    uint64_t idx = 0;
    for (int i = 0; i < n; ++i) idx = (idx << 1) | batch.configs(b, i);
    ++counts[idx];
  }
  // goodness_of_fit (oracle.cpp:132-178)
  double tv = 0.0, chi = 0.0, pe = 0.0, po = 0.0;
  long bins = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const double p = std::exp(lp[i]);
    tv += std::fabs(p - (double)counts[i] / (double)samples);
    const double e = p * (double)samples;
    if (e < 5.0) {
      pe += e;
      po += (double)counts[i];
      continue;
    }
    chi += ((double)counts[i] - e) * ((double)counts[i] - e) / e;
    ++bins;
  }
  tv *= 0.5;
  if (pe > 0.0) {
    chi += (po - pe) * (po - pe) / pe;
    ++bins;
  }
  const long dof = std::max(1L, bins - 1);
  const double k = (double)dof;
  const double z = (std::cbrt(chi / k) - (1.0 - 2.0 / (9.0 * k))) / std::sqrt(2.0 / (9.0 * k));
  std::cout << "samples " << samples << "\n";
  std::cout << "tv_distance " << tv << "\n";
  std::cout << "chi_square " << chi << " dof " << dof << " z " << z << "\n";
  const bool reject = tv > 0.02 || z > 3.090232;
  std::cout << (reject ? "REJECT" : "PASS") << "\n";
  return reject ? kExitRejected : 0;
}

int run_gen(const Args& a) {  // gen-instance (vqmc.cpp:469-488)
  if (!a.has("problem") || !a.has("n") || !a.has("out")) throw UsageError("--problem, --n and --out are required");
  const std::string problem = a.get("problem", "");
  if (problem != "tim" && problem != "maxcut") throw UsageError("--problem: not in {tim, maxcut}");
  const std::string out = a.get("out", "");
  const int n = (int)a.geti("n", 0);
  const uint64_t seed = (uint64_t)a.geti("seed", 0);
  if (problem == "tim") vqmc::save_spec(vqmc::random_tim(n, seed), out);  // vqmc.cpp:478-481
  else vqmc::save_graph(vqmc::random_maxcut_graph(n, seed), out);
  std::cout << "wrote " << out << "\n";
  return 0;
}

void usage() {
  std::cout << "vqmc (B200): variational Monte Carlo (Max-Cut, TIM) with MADE + AUTO + ADAM / SGD + SR\n"
               "subcommands: solve | oracle | sample-test | gen-instance\n";
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  if (args.empty()) {
    usage();
    std::cerr << "A subcommand is required\n";
    return kExitUsage;
  }
  const std::string cmd = args.front();
  args.erase(args.begin());
  if (cmd == "--help" || cmd == "-h") {
    usage();
    return 0;
  }
  try {
    if (cmd == "solve") {
      std::string config;  // splice --config entries first so explicit flags win
      for (size_t i = 0; i < args.size(); ++i) {
        if (args[i] == "--config" && i + 1 < args.size()) config = args[i + 1];
        if (args[i].rfind("--config=", 0) == 0) config = args[i].substr(9);
      }
      if (!config.empty()) {
        const auto extra = config_file_args(config);
        args.insert(args.begin(), extra.begin(), extra.end());
      }
      const Args a = parse(args,
                           {"config", "instance", "problem", "n", "seed", "model", "sampler", "hidden", "chains",
                            "burn-in", "thinning", "optimizer", "lr", "sr-lambda", "sr-tol", "sr-maxiter",
                            "iterations", "minibatch", "eval-batch", "workers", "target", "out", "save-model",
                            "device", "gpus"},
                           {"mcmc-reburn", "sr-fallback", "sr-uncentered", "reference-streams"});
      return run_solve(a);
    }
    if (cmd == "oracle") return run_oracle(parse(args, {"instance"}, {}));
    if (cmd == "sample-test")
      return run_sample_test(parse(args, {"checkpoint", "model", "n", "hidden", "samples", "seed", "chains",
                                          "burn-in", "thinning"},
                                   {}));
    if (cmd == "gen-instance") return run_gen(parse(args, {"problem", "n", "seed", "out"}, {}));
    if (cmd == "benchmark") throw UsageError("benchmark (TIM weak scaling) is outside the B200 path; use bench.py");
    throw UsageError("unknown subcommand: " + cmd);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return kExitNumerical;
  }
}
