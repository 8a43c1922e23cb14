// speig_cli.cpp — `flz-speig`: the reference's command-line front end (tools/speig_main.cpp)
// over the B200 solver, same subcommands, flags, report schema and exit codes, so that scripts
// written against `speig` keep working:
//
//   flz-speig solve       --matrix A.mtx --lo a --hi b [--block r] [--degree m] [--epsilon e]
//                         [--tol t] [--max-dim d] [--seed s] [--check-every k] [--plain]
//                         [--out report.json] [--vectors V.mtx]
//   flz-speig filter-info --lo a --hi b [--degree m] [--epsilon e] [--bounds lo,hi]
//                         [--samples n] [--json]            (host only: needs no GPU)
//   flz-speig info        --matrix A.mtx [--bounds-steps k]
//   flz-speig bench       --matrix A.mtx --lo a --hi b --degrees 30,60,auto [...solve flags]
//                         [--csv rows.csv] [--out rows.json]
//
// Exit codes (speig_main.cpp:21-24): 0 ok, 1 usage / parse / file errors, 2 invalid interval,
// 3 not converged within max_dim (the partial report is still written).  Report keys follow
// speig_main.cpp:59-91 (an object with alphabetically ordered keys, two-space indent — what
// the reference's JSON library emits).  The reference uses CLI11 and nlohmann/json, neither of
// which is vendored here; the option tables and the JSON writer below are this file's own.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <variant>
#include <vector>

#include "flz/solver.hpp"

namespace {

enum Exit { kOk = 0, kUsage = 1, kInterval = 2, kUnconverged = 3 };

// ----------------------------------------------------------------------------- JSON
class Json {
 public:
  using Array = std::vector<Json>;
  using Object = std::map<std::string, Json>;   // ordered keys, like the reference's reports
  Json() : v_(nullptr) {}
  Json(bool b) : v_(b) {}
  Json(int i) : v_((std::int64_t)i) {}
  Json(std::int64_t i) : v_(i) {}
  Json(std::uint64_t u) : v_(u) {}
  Json(std::size_t u, int) : v_((std::uint64_t)u) {}
  Json(double d) : v_(d) {}
  Json(const char* s) : v_(std::string(s)) {}
  Json(std::string s) : v_(std::move(s)) {}
  Json(Array a) : v_(std::move(a)) {}
  Json(Object o) : v_(std::move(o)) {}
  static Json numbers(const std::vector<double>& xs) {
    Array a;
    for (double x : xs) a.emplace_back(x);
    return Json(std::move(a));
  }
  Json& operator[](const std::string& key) {
    if (!std::holds_alternative<Object>(v_)) v_ = Object{};
    return std::get<Object>(v_)[key];
  }
  void push_back(Json x) {
    if (!std::holds_alternative<Array>(v_)) v_ = Array{};
    std::get<Array>(v_).push_back(std::move(x));
  }
  std::string dump(int indent) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  static void number(std::string& out, double d) {
    if (!std::isfinite(d)) {   // JSON has no inf/nan
      out += "null";
      return;
    }
    char buf[40];
    auto r = std::to_chars(buf, buf + sizeof buf, d);   // shortest text that round-trips
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eE") == std::string::npos) s += ".0";
    out += s;
  }
  static void quoted(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\n': out += "\\n"; break;
        case '\r': out += "\\r"; break;
        case '\t': out += "\\t"; break;
        default:
          if (c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", c);
            out += b;
          } else {
            out += (char)c;
          }
      }
    }
    out += '"';
  }
  void write(std::string& out, int indent, int depth) const {
    const std::string pad((size_t)indent * (depth + 1), ' '), close((size_t)indent * depth, ' ');
    std::visit(
        [&](const auto& x) {
          using T = std::decay_t<decltype(x)>;
          if constexpr (std::is_same_v<T, std::nullptr_t>) out += "null";
          else if constexpr (std::is_same_v<T, bool>) out += x ? "true" : "false";
          else if constexpr (std::is_same_v<T, std::int64_t> || std::is_same_v<T, std::uint64_t>)
            out += std::to_string(x);
          else if constexpr (std::is_same_v<T, double>) number(out, x);
          else if constexpr (std::is_same_v<T, std::string>) quoted(out, x);
          else if constexpr (std::is_same_v<T, Array>) {
            if (x.empty()) {
              out += "[]";
              return;
            }
            out += "[\n";
            for (size_t i = 0; i < x.size(); ++i) {
              out += pad;
              x[i].write(out, indent, depth + 1);
              out += i + 1 < x.size() ? ",\n" : "\n";
            }
            out += close + "]";
          } else {
            if (x.empty()) {
              out += "{}";
              return;
            }
            out += "{\n";
            size_t i = 0;
            for (const auto& [k, v] : x) {
              out += pad;
              quoted(out, k);
              out += ": ";
              v.write(out, indent, depth + 1);
              out += ++i < x.size() ? ",\n" : "\n";
            }
            out += close + "}";
          }
        },
        v_);
  }
  std::variant<std::nullptr_t, bool, std::int64_t, std::uint64_t, double, std::string, Array, Object> v_;
};

// ------------------------------------------------------------------- option tables
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Option {
  std::string name;   // "--matrix"
  std::string help;
  bool required = false;
  bool flag = false;  // takes no value
  int values = 1;     // values it consumes (--bounds: 2, also as "lo,hi")
  std::function<void(const std::vector<std::string>&)> store;
  bool seen = false;
};

template <class T>
T parse_number(const std::string& opt, const std::string& text) {
  T v{};
  const char* b = text.data();
  const char* e = b + text.size();
  if (b != e && *b == '+') ++b;
  std::from_chars_result r{};
  if constexpr (std::is_floating_point_v<T>) r = std::from_chars(b, e, v);
  else r = std::from_chars(b, e, v, 10);
  if (r.ec != std::errc() || r.ptr != e)
    throw UsageError(opt + ": '" + text + "' is not a valid " +
                     (std::is_floating_point_v<T> ? "number" : "integer"));
  return v;
}

class Command {
 public:
  Command(std::string name, std::string help) : name_(std::move(name)), help_(std::move(help)) {}
  template <class T>
  Command& value(const std::string& opt, T& target, const std::string& help, bool required = false) {
    Option o;
    o.name = opt;
    o.help = help;
    o.required = required;
    if constexpr (std::is_same_v<T, std::string>)
      o.store = [&target](const std::vector<std::string>& v) { target = v[0]; };
    else
      o.store = [&target, opt](const std::vector<std::string>& v) { target = parse_number<T>(opt, v[0]); };
    opts_.push_back(std::move(o));
    return *this;
  }
  Command& flag(const std::string& opt, bool& target, const std::string& help) {
    Option o;
    o.name = opt;
    o.help = help;
    o.flag = true;
    o.values = 0;
    o.store = [&target](const std::vector<std::string>&) { target = true; };
    opts_.push_back(std::move(o));
    return *this;
  }
  Command& pair(const std::string& opt, std::vector<double>& target, const std::string& help) {
    Option o;
    o.name = opt;
    o.help = help;
    o.values = 2;
    o.store = [&target, opt](const std::vector<std::string>& v) {
      target = {parse_number<double>(opt, v[0]), parse_number<double>(opt, v[1])};
    };
    opts_.push_back(std::move(o));
    return *this;
  }
  const std::string& name() const { return name_; }
  const std::string& help() const { return help_; }

  // argv after the subcommand name; returns false when --help was asked for (help printed)
  bool parse(const std::vector<std::string>& args) {
    for (size_t i = 0; i < args.size(); ++i) {
      std::string a = args[i];
      if (a == "-h" || a == "--help") {
        print_help(std::cout);
        return false;
      }
      std::optional<std::string> inline_value;
      if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
        inline_value = a.substr(eq + 1);
        a = a.substr(0, eq);
      }
      auto it = std::find_if(opts_.begin(), opts_.end(), [&](const Option& o) { return o.name == a; });
      if (it == opts_.end()) throw UsageError("unknown argument '" + args[i] + "' for " + name_);
      std::vector<std::string> vals;
      if (it->flag) {
        if (inline_value) throw UsageError(a + " takes no value");
      } else {
        std::string first;
        if (inline_value) first = *inline_value;
        else if (i + 1 < args.size()) first = args[++i];
        else throw UsageError(a + " expects a value");
        if (it->values == 2) {   // "lo,hi" or "lo hi"
          if (const auto comma = first.find(','); comma != std::string::npos) {
            vals = {first.substr(0, comma), first.substr(comma + 1)};
          } else {
            if (i + 1 >= args.size()) throw UsageError(a + " expects two values lo,hi");
            vals = {first, args[++i]};
          }
        } else {
          vals = {first};
        }
      }
      it->store(vals);
      it->seen = true;
    }
    for (const Option& o : opts_)
      if (o.required && !o.seen) throw UsageError(o.name + " is required");
    return true;
  }
  void print_help(std::ostream& os) const {
    os << "flz-speig " << name_ << " — " << help_ << "\n\noptions:\n";
    for (const Option& o : opts_) {
      std::string left = "  " + o.name + (o.flag ? "" : (o.values == 2 ? " LO,HI" : " VALUE"));
      if (left.size() < 26) left.resize(26, ' ');
      os << left << o.help << (o.required ? "  (required)" : "") << "\n";
    }
  }

 private:
  std::string name_, help_;
  std::vector<Option> opts_;
};

// ----------------------------------------------------------------------------- solve
struct SolveOptions {
  std::string matrix;
  double lo = 0.0, hi = 0.0;
  int block = 3;
  int degree = 0;   // 0 = automatic
  double epsilon = flz::kDefaultFilterEpsilon;
  double tol = 1e-10;
  int max_dim = 0;
  std::uint64_t seed = 20177;
  int check_every = 10;
  bool plain = false;
  std::string out, vectors;

  flz::LanczosConfig config() const {
    flz::LanczosConfig c;
    c.block_size = block;
    c.tol = tol;
    c.max_dim = max_dim;
    c.seed = seed;
    c.check_every = check_every;
    c.epsilon = epsilon;
    if (degree > 0) c.degree = degree;
    return c;
  }
  void declare(Command& cmd, bool with_degree) {
    cmd.value("--matrix", matrix, "Matrix Market file", true)
        .value("--lo", lo, "interval lower endpoint", true)
        .value("--hi", hi, "interval upper endpoint", true)
        .value("--block", block, "Lanczos block size (default 3)");
    if (with_degree) cmd.value("--degree", degree, "fixed filter degree (default: auto)");
    cmd.value("--epsilon", epsilon, "auto-degree tolerance")
        .value("--tol", tol, "relative residual tolerance")
        .value("--max-dim", max_dim, "basis size cap (default min(n, 3000))")
        .value("--seed", seed, "random seed")
        .value("--check-every", check_every, "blocks between convergence checks")
        .flag("--plain", plain, "iterate with A itself (no filter)");
  }
};

double share(double part, double total) {
  return total > 0.0 ? std::clamp(100.0 * part / total, 0.0, 100.0) : 0.0;
}
double worst(const std::vector<double>& residuals) {
  double m = 0.0;
  for (double r : residuals) m = std::max(m, r);
  return m;
}

Json report(const SolveOptions& opt, const flz::EigenResult& res, const flz::LanczosConfig& cfg) {
  const flz::SolveStats& s = res.stats;
  Json j;
  j["matrix"] = opt.matrix;
  j["interval"] = Json::numbers({opt.lo, opt.hi});
  j["eigs"] = Json(res.eigenvalues.size(), 0);
  j["degree"] = s.degree;
  j["iters"] = s.block_steps;
  j["basis_vectors"] = s.basis_vectors;
  j["mv"] = s.mv_iteration;
  j["mv_bounds"] = s.mv_bounds;
  j["mv_total"] = s.mv_total;
  j["time_s"] = s.time_total_s;
  j["max_residual"] = worst(res.residuals);
  j["preproc_pct"] = share(s.time_preproc_s, s.time_total_s);
  j["orth_pct"] = share(s.time_orth_s, s.time_total_s);
  j["mv_pct"] = share(s.time_mv_s, s.time_total_s);
  j["converged"] = s.converged;
  j["eigenvalues"] = Json::numbers(res.eigenvalues);
  Json c;
  c["block"] = cfg.block_size;
  c["tol"] = cfg.tol;
  c["max_dim"] = cfg.max_dim;
  c["seed"] = cfg.seed;
  c["check_every"] = cfg.check_every;
  c["epsilon"] = cfg.epsilon;
  c["degree"] = cfg.degree ? Json(*cfg.degree) : Json("auto");
  c["plain"] = opt.plain;
  j["config"] = std::move(c);
  return j;
}

int write_text(const std::string& path, const std::string& text) {
  std::ofstream out(path);
  if (!out) {
    std::cerr << "error: cannot write '" << path << "'\n";
    return kUsage;
  }
  out << text;
  return kOk;
}

flz::EigenResult run_solver(const flz::SparseSymMatrix& A, const SolveOptions& opt,
                            const flz::LanczosConfig& cfg) {
  return opt.plain ? flz::plain_lanczos(A, opt.lo, opt.hi, cfg)
                   : flz::filtered_lanczos(A, opt.lo, opt.hi, cfg);
}

int cmd_solve(const SolveOptions& opt) {
  const flz::SparseSymMatrix A = flz::load_matrix_market(opt.matrix);
  const flz::LanczosConfig cfg = opt.config();
  const flz::EigenResult res = run_solver(A, opt, cfg);   // IntervalError -> exit 2 in main
  if (!opt.out.empty())
    if (int rc = write_text(opt.out, report(opt, res, cfg).dump(2) + "\n"); rc != kOk) return rc;
  if (!opt.vectors.empty()) flz::save_dense_matrix_market(res.eigenvectors, opt.vectors);

  const flz::SolveStats& s = res.stats;
  std::printf("matrix        %s (n=%zu, nnz=%zu)\n", opt.matrix.c_str(), A.dim(), A.nnz());
  std::printf("interval      [%.17g, %.17g]%s\n", opt.lo, opt.hi, opt.plain ? "  (plain)" : "");
  if (!opt.plain) std::printf("degree        %d%s\n", s.degree, s.degree_clamped ? "  (clamped)" : "");
  std::printf("iters         %d  (basis vectors: %d)\n", s.block_steps, s.basis_vectors);
  std::printf("MV            %llu  (+%llu for bounds)\n", (unsigned long long)s.mv_iteration,
              (unsigned long long)s.mv_bounds);
  std::printf("time          %.3fs  (preproc %.1f%%, orth %.1f%%, mv %.1f%%)\n", s.time_total_s,
              share(s.time_preproc_s, s.time_total_s), share(s.time_orth_s, s.time_total_s),
              share(s.time_mv_s, s.time_total_s));
  std::printf("max residual  %.3e\n", worst(res.residuals));
  std::printf("eigenvalues   %zu\n", res.eigenvalues.size());
  for (double v : res.eigenvalues) std::printf("%.17g\n", v);
  if (!s.converged) {
    std::cerr << "warning: not converged within max_dim=" << cfg.resolved_max_dim(A.dim())
              << " basis vectors\n";
    return kUnconverged;
  }
  return kOk;
}

// ----------------------------------------------------------------------- filter-info
struct FilterInfoOptions {
  double lo = 0.0, hi = 0.0;
  int degree = 0;
  double epsilon = flz::kDefaultFilterEpsilon;
  std::vector<double> bounds{-1.0, 1.0};
  int samples = 2001;
  bool json = false;
};

int cmd_filter_info(const FilterInfoOptions& opt) {
  const flz::SpectralBounds bounds(opt.bounds[0], opt.bounds[1]);
  const flz::ChebyshevFilter f = flz::build_filter(
      bounds, opt.lo, opt.hi, opt.degree > 0 ? std::optional<int>(opt.degree) : std::nullopt,
      opt.epsilon);
  const int ns = std::max(2, opt.samples);
  const double width = bounds.lambda_max() - bounds.lambda_min();
  std::vector<double> x(ns), y(ns);
  for (int i = 0; i < ns; ++i) {
    x[i] = bounds.lambda_min() + width * i / (ns - 1);
    y[i] = f.evaluate(x[i]);
  }
  const auto coeffs = f.coefficients();
  if (opt.json) {
    Json j;
    j["degree"] = f.degree();
    j["clamped"] = f.degree_clamped();
    j["interval"] = Json::numbers({f.alpha(), f.beta()});
    j["bounds"] = Json::numbers({bounds.lambda_min(), bounds.lambda_max()});
    j["coefficients"] = Json::numbers(std::vector<double>(coeffs.begin(), coeffs.end()));
    Json pts{Json::Array{}};
    for (int i = 0; i < ns; ++i) pts.push_back(Json::numbers({x[i], y[i]}));
    j["samples"] = std::move(pts);
    std::cout << j.dump(2) << "\n";
    return kOk;
  }
  std::printf("# degree,%d\n", f.degree());
  if (f.degree_clamped()) std::printf("# clamped,1\n");
  std::printf("# alpha,%.17g\n# beta,%.17g\n", f.alpha(), f.beta());
  std::printf("# bounds,%.17g,%.17g\n", bounds.lambda_min(), bounds.lambda_max());
  std::printf("record,x,value\n");
  for (size_t i = 0; i < coeffs.size(); ++i) std::printf("coef,%zu,%.17g\n", i, coeffs[i]);
  for (int i = 0; i < ns; ++i) std::printf("sample,%.17g,%.17g\n", x[i], y[i]);
  return kOk;
}

// ------------------------------------------------------------------------------ info
int cmd_info(const std::string& matrix, int steps) {
  const flz::SparseSymMatrix A = flz::load_matrix_market(matrix);
  std::printf("matrix    %s\n", matrix.c_str());
  std::printf("n         %zu\n", A.dim());
  std::printf("nnz       %zu\n", A.nnz());
  std::printf("nnz/n     %.1f\n", A.dim() ? (double)A.nnz() / (double)A.dim() : 0.0);
  std::printf("kernels   sm_100a (libflz)\n");
  try {
    const flz::SpectralBounds b = flz::estimate_spectral_bounds(A, steps);
    std::printf("spectral interval  [%.6g, %.6g]  (estimated, %d Lanczos steps)\n", b.lambda_min(),
                b.lambda_max(), steps);
  } catch (const flz::Error& e) {
    std::printf("spectral interval  unavailable (%s)\n", e.what());
  }
  return kOk;
}

// ----------------------------------------------------------------------------- bench
struct BenchOptions {
  SolveOptions base;
  std::string degrees = "auto", csv, out;
};

int cmd_bench(const BenchOptions& opt) {
  const flz::SparseSymMatrix A = flz::load_matrix_market(opt.base.matrix);
  std::vector<std::string> labels;
  {
    std::string tok;
    for (char c : opt.degrees + ",") {
      if (c == ',') {
        if (!tok.empty()) labels.push_back(tok);
        tok.clear();
      } else if (!std::isspace((unsigned char)c)) {
        tok += c;
      }
    }
  }
  if (labels.empty()) {
    std::cerr << "error: --degrees expects a comma-separated list (integers or 'auto')\n";
    return kUsage;
  }
  struct Row {
    std::string label, error;
    bool solved = false, failed = false;
    flz::EigenResult res;
    flz::LanczosConfig cfg;
  };
  std::vector<Row> rows;
  for (const std::string& label : labels) {
    SolveOptions one = opt.base;
    if (label == "auto") {
      one.degree = 0;
    } else {
      int m = 0;
      const auto r = std::from_chars(label.data(), label.data() + label.size(), m);
      if (r.ec != std::errc() || r.ptr != label.data() + label.size()) {
        std::cerr << "error: bad degree '" << label << "'\n";
        return kUsage;
      }
      if (m < 1) {
        std::cerr << "error: degree must be >= 1\n";
        return kUsage;
      }
      one.degree = m;
    }
    Row row;
    row.label = label;
    row.cfg = one.config();
    try {
      row.res = run_solver(A, one, row.cfg);
      row.solved = true;
      if (!row.res.stats.converged) {
        row.failed = true;
        row.error = "not converged";
      }
    } catch (const flz::Error& e) {
      row.failed = true;
      row.error = e.what();
    }
    rows.push_back(std::move(row));
  }
  const bool all_ok = std::none_of(rows.begin(), rows.end(), [](const Row& r) { return r.failed; });

  std::printf("%-8s %6s %6s %10s %10s %12s %7s %7s %7s  %s\n", "degree", "eigs", "iters", "MV",
              "time(s)", "residual", "PRE%", "ORTH%", "MV%", "status");
  for (const Row& r : rows) {
    if (!r.solved) {
      std::printf("%-8s %6s %6s %10s %10s %12s %7s %7s %7s  error: %s\n", r.label.c_str(), "-", "-",
                  "-", "-", "-", "-", "-", "-", r.error.c_str());
      continue;
    }
    const flz::SolveStats& s = r.res.stats;
    std::printf("%-8d %6zu %6d %10llu %10.3f %12.3e %7.1f %7.1f %7.1f  %s\n", s.degree,
                r.res.eigenvalues.size(), s.block_steps, (unsigned long long)s.mv_iteration,
                s.time_total_s, worst(r.res.residuals), share(s.time_preproc_s, s.time_total_s),
                share(s.time_orth_s, s.time_total_s), share(s.time_mv_s, s.time_total_s),
                r.failed ? r.error.c_str() : "ok");
  }
  if (!opt.csv.empty()) {
    std::string csv =
        "matrix,lo,hi,eigs,degree,iters,mv,time_s,max_residual,preproc_pct,orth_pct,mv_pct,converged\n";
    char buf[640];
    for (const Row& r : rows) {
      if (!r.solved) {
        std::snprintf(buf, sizeof buf, "%s,%.17g,%.17g,,,,,,,,,,error\n", opt.base.matrix.c_str(),
                      opt.base.lo, opt.base.hi);
      } else {
        const flz::SolveStats& s = r.res.stats;
        std::snprintf(buf, sizeof buf, "%s,%.17g,%.17g,%zu,%d,%d,%llu,%.6g,%.6g,%.6g,%.6g,%.6g,%s\n",
                      opt.base.matrix.c_str(), opt.base.lo, opt.base.hi, r.res.eigenvalues.size(),
                      s.degree, s.block_steps, (unsigned long long)s.mv_iteration, s.time_total_s,
                      worst(r.res.residuals), share(s.time_preproc_s, s.time_total_s),
                      share(s.time_orth_s, s.time_total_s), share(s.time_mv_s, s.time_total_s),
                      s.converged ? "true" : "false");
      }
      csv += buf;
    }
    if (int rc = write_text(opt.csv, csv); rc != kOk) return rc;
  }
  if (!opt.out.empty()) {
    Json all{Json::Array{}};
    for (const Row& r : rows) {
      if (!r.solved) {
        Json e;
        e["degree"] = r.label;
        e["error"] = r.error;
        all.push_back(std::move(e));
      } else {
        SolveOptions one = opt.base;
        all.push_back(report(one, r.res, r.cfg));
      }
    }
    if (int rc = write_text(opt.out, all.dump(2) + "\n"); rc != kOk) return rc;
  }
  return all_ok ? kOk : kUnconverged;
}

void print_top_help(const std::vector<Command*>& cmds, std::ostream& os) {
  os << "flz-speig — interval eigenvalues of sparse symmetric matrices (filtered block Lanczos, "
        "B200)\n\nusage: flz-speig SUBCOMMAND [options]\n\nsubcommands:\n";
  for (const Command* c : cmds) {
    std::string left = "  " + c->name();
    left.resize(16, ' ');
    os << left << c->help() << "\n";
  }
  os << "\n`flz-speig SUBCOMMAND --help` lists the options of a subcommand.\n";
}

}  // namespace

int main(int argc, char** argv) {
  SolveOptions solve_opt;
  Command solve("solve", "compute all eigenpairs in [lo, hi]");
  solve_opt.declare(solve, true);
  solve.value("--out", solve_opt.out, "write a JSON report here")
      .value("--vectors", solve_opt.vectors, "write eigenvectors (MM array format)");

  FilterInfoOptions fi_opt;
  Command fi("filter-info", "dump a filter's coefficients and samples");
  fi.value("--lo", fi_opt.lo, "interval lower endpoint", true)
      .value("--hi", fi_opt.hi, "interval upper endpoint", true)
      .value("--degree", fi_opt.degree, "fixed degree (default: auto)")
      .value("--epsilon", fi_opt.epsilon, "auto-degree tolerance")
      .pair("--bounds", fi_opt.bounds, "spectral bounds lo,hi (default -1,1)")
      .value("--samples", fi_opt.samples, "evaluation grid size (default 2001)")
      .flag("--json", fi_opt.json, "emit JSON instead of CSV");

  std::string info_matrix;
  int info_steps = 50;
  Command info("info", "matrix summary and estimated spectral interval");
  info.value("--matrix", info_matrix, "Matrix Market file", true)
      .value("--bounds-steps", info_steps, "Lanczos steps for the estimate");

  BenchOptions bench_opt;
  Command bench("bench", "one solve per filter degree, tabulated");
  bench_opt.base.declare(bench, false);
  bench.value("--degrees", bench_opt.degrees, "comma-separated degrees; 'auto' selects automatically", true)
      .value("--csv", bench_opt.csv, "write rows as CSV here")
      .value("--out", bench_opt.out, "write rows as JSON here");

  const std::vector<Command*> cmds{&solve, &fi, &info, &bench};
  if (argc < 2) {
    print_top_help(cmds, std::cerr);
    return kUsage;
  }
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    print_top_help(cmds, std::cout);
    return kOk;
  }
  const auto it = std::find_if(cmds.begin(), cmds.end(), [&](const Command* c) { return c->name() == sub; });
  if (it == cmds.end()) {
    std::cerr << "error: unknown subcommand '" << sub << "'\n";
    print_top_help(cmds, std::cerr);
    return kUsage;
  }
  try {
    if (!(*it)->parse(std::vector<std::string>(argv + 2, argv + argc))) return kOk;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\nrun `flz-speig " << sub << " --help` for the options\n";
    return kUsage;
  }
  try {
    if (*it == &solve) return cmd_solve(solve_opt);
    if (*it == &fi) return cmd_filter_info(fi_opt);
    if (*it == &info) return cmd_info(info_matrix, info_steps);
    return cmd_bench(bench_opt);
  } catch (const flz::IntervalError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kInterval;
  } catch (const std::exception& e) {   // flz::Error (parse, file, device) and anything else
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  }
}
