// tsieve -- command-line front end of the B200 drop-in.
//
// Same subcommands, flags, record fields and exit codes as the reference CLI
// (/root/reference/proj/tools/main.cpp: exit codes :27-30, flags :32-81,
// load_instance :126-231, record_json :251-291, print_record :293-329,
// run_solver_command :331-341, run_verify :414-441, main :645-727) for
// decide / extract / optimum / verify.  `gen` and `bench` belong to the
// reference's own benchmark harness and are replaced by bench.py.
//
// Exit status: 0 = YES, 1 = NO, 2 = usage or input error, 3 = extraction
// failure.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <variant>
#include <vector>

#include "tsieve/solver.hpp"

using namespace tsieve;

namespace {

constexpr int kYes = 0, kNo = 1, kUsage = 2, kBudget = 3;

struct UsageError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// ---- minimal JSON value (writer + reader) --------------------------------

struct Json {
  using Obj = std::map<std::string, Json>;  // sorted keys, like the reference's dump
  using Arr = std::vector<Json>;
  std::variant<std::nullptr_t, bool, double, std::int64_t, std::string, Arr, Obj> v;
  Json() : v(nullptr) {}
  Json(std::nullptr_t) : v(nullptr) {}
  Json(bool b) : v(b) {}
  Json(int x) : v(static_cast<std::int64_t>(x)) {}
  Json(std::int64_t x) : v(x) {}
  Json(std::uint64_t x) : v(static_cast<std::int64_t>(x)) {}
  Json(double x) : v(x) {}
  Json(const char* s) : v(std::string(s)) {}
  Json(std::string s) : v(std::move(s)) {}
  Json(Arr a) : v(std::move(a)) {}
  Json(Obj o) : v(std::move(o)) {}

  const Json* get(const std::string& k) const {
    if (auto* o = std::get_if<Obj>(&v)) {
      auto it = o->find(k);
      if (it != o->end()) return &it->second;
    }
    return nullptr;
  }
  bool is_null() const { return std::holds_alternative<std::nullptr_t>(v); }
  std::int64_t as_int() const {
    if (auto* i = std::get_if<std::int64_t>(&v)) return *i;
    if (auto* d = std::get_if<double>(&v)) return static_cast<std::int64_t>(*d);
    throw std::invalid_argument("witness file: expected an integer");
  }
  const Arr& as_arr() const {
    if (auto* a = std::get_if<Arr>(&v)) return *a;
    throw std::invalid_argument("witness file: expected an array");
  }
};

void quote(std::ostream& os, const std::string& s) {
  os << '"';
  for (char c : s) {
    if (c == '"' || c == '\\') os << '\\' << c;
    else if (c == '\n') os << "\\n";
    else os << c;
  }
  os << '"';
}

void dump(std::ostream& os, const Json& j, int indent) {
  const std::string pad(static_cast<size_t>(indent) * 2, ' ');
  const std::string in(static_cast<size_t>(indent + 1) * 2, ' ');
  std::visit(
      [&](const auto& x) {
        using T = std::decay_t<decltype(x)>;
        if constexpr (std::is_same_v<T, std::nullptr_t>) {
          os << "null";
        } else if constexpr (std::is_same_v<T, bool>) {
          os << (x ? "true" : "false");
        } else if constexpr (std::is_same_v<T, std::int64_t>) {
          os << x;
        } else if constexpr (std::is_same_v<T, double>) {
          char b[64];
          std::snprintf(b, sizeof b, "%.17g", x);
          os << b;
        } else if constexpr (std::is_same_v<T, std::string>) {
          quote(os, x);
        } else if constexpr (std::is_same_v<T, Json::Arr>) {
          if (x.empty()) {
            os << "[]";
            return;
          }
          os << "[\n";
          for (size_t i = 0; i < x.size(); ++i) {
            os << in;
            dump(os, x[i], indent + 1);
            os << (i + 1 < x.size() ? ",\n" : "\n");
          }
          os << pad << "]";
        } else {
          if (x.empty()) {
            os << "{}";
            return;
          }
          os << "{\n";
          size_t i = 0;
          for (const auto& [k, val] : x) {
            os << in;
            quote(os, k);
            os << ": ";
            dump(os, val, indent + 1);
            os << (++i < x.size() ? ",\n" : "\n");
          }
          os << pad << "}";
        }
      },
      j.v);
}

class Reader {
 public:
  explicit Reader(std::string s) : s_(std::move(s)) {}
  Json parse() {
    Json j = value();
    ws();
    return j;
  }

 private:
  void ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  [[noreturn]] void bad() { throw std::invalid_argument("witness file: malformed JSON"); }
  bool eat(const char* lit) {
    const size_t n = std::char_traits<char>::length(lit);
    if (s_.compare(i_, n, lit) != 0) return false;
    i_ += n;
    return true;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) bad();
    const char c = s_[i_];
    if (c == '{') {
      ++i_;
      Json::Obj o;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') {
        ++i_;
        return o;
      }
      for (;;) {
        ws();
        Json key = value();
        auto* ks = std::get_if<std::string>(&key.v);
        if (!ks) bad();
        ws();
        if (i_ >= s_.size() || s_[i_++] != ':') bad();
        o[*ks] = value();
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == '}') {
          ++i_;
          return o;
        }
        bad();
      }
    }
    if (c == '[') {
      ++i_;
      Json::Arr a;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') {
        ++i_;
        return a;
      }
      for (;;) {
        a.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == ']') {
          ++i_;
          return a;
        }
        bad();
      }
    }
    if (c == '"') {
      ++i_;
      std::string out;
      while (i_ < s_.size() && s_[i_] != '"') {
        if (s_[i_] == '\\' && i_ + 1 < s_.size()) ++i_;
        out += s_[i_++];
      }
      if (i_ >= s_.size()) bad();
      ++i_;
      return out;
    }
    if (eat("true")) return true;
    if (eat("false")) return false;
    if (eat("null")) return nullptr;
    size_t used = 0;
    const std::string rest = s_.substr(i_, 64);
    try {
      if (rest.find_first_of(".eE") < rest.find_first_of(",]} \n\t\r")) {
        const double d = std::stod(rest, &used);
        i_ += used;
        return d;
      }
      const long long x = std::stoll(rest, &used);
      i_ += used;
      return static_cast<std::int64_t>(x);
    } catch (const std::exception&) {
      bad();
    }
  }
  std::string s_;
  size_t i_ = 0;
};

// ---- flags ---------------------------------------------------------------

struct Opts {
  std::string graph_file, colors_file, delays_file;
  std::string ingest_cache;  // binary ingest cache of --graph ("" = none); not a reference flag
  std::string problem = "pathmotif";
  std::string motif, order, times;
  int k = 0;
  std::string source, dest;
  std::uint64_t seed = 1;
  int field_bits = 64;
  int lanes = 8;
  int threads = 0;
  std::string preprocess = "both";
  std::string extraction = "localized";
  std::string edge_model = "auto";
  int wildcards_max = 0;
  bool directed = false;
  std::string format = "text";
  bool optimize = true;
  std::string witness_file;
  int device = 0;
};

long long to_int(const std::string& flag, const std::string& val) {
  size_t used = 0;
  long long x = 0;
  try {
    x = std::stoll(val, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != val.size())
    throw UsageError(flag + ": invalid integer '" + val + "'");
  return x;
}

Opts parse_flags(const std::string& cmd, int argc, char** argv) {
  Opts o;
  bool have_graph = false, have_witness = false;
  for (int i = 0; i < argc; ++i) {
    const std::string f = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw UsageError(f + " requires an argument");
      return argv[++i];
    };
    if (f == "--graph") o.graph_file = val(), have_graph = true;
    else if (f == "--colors") o.colors_file = val();
    else if (f == "--ingest-cache") o.ingest_cache = val();
    else if (f == "--delays") o.delays_file = val();
    else if (f == "--problem") o.problem = val();
    else if (f == "--motif") o.motif = val();
    else if (f == "--order") o.order = val();
    else if (f == "--times") o.times = val();
    else if (f == "--k") o.k = static_cast<int>(to_int(f, val()));
    else if (f == "--source") o.source = val();
    else if (f == "--dest") o.dest = val();
    else if (f == "--seed") o.seed = static_cast<std::uint64_t>(to_int(f, val()));
    else if (f == "--field-bits") o.field_bits = static_cast<int>(to_int(f, val()));
    else if (f == "--lanes") o.lanes = static_cast<int>(to_int(f, val()));
    else if (f == "--threads") o.threads = static_cast<int>(to_int(f, val()));
    else if (f == "--preprocess") o.preprocess = val();
    else if (f == "--extraction") o.extraction = val();
    else if (f == "--edge-model") o.edge_model = val();
    else if (f == "--wildcards-max") o.wildcards_max = static_cast<int>(to_int(f, val()));
    else if (f == "--directed") o.directed = true;
    else if (f == "--format") o.format = val();
    else if (f == "--device") o.device = static_cast<int>(to_int(f, val()));
    else if (cmd == "extract" && f == "--optimize") o.optimize = true;
    else if (cmd == "extract" && f == "--no-optimize") o.optimize = false;
    else if (cmd == "verify" && f == "--witness") o.witness_file = val(), have_witness = true;
    else throw UsageError("The following argument was not expected: " + f);
  }
  if (!have_graph) throw UsageError("--graph is required");
  if (cmd == "verify" && !have_witness) throw UsageError("--witness is required");
  if (o.format != "text" && o.format != "json")
    throw UsageError("--format: unknown '" + o.format + "'");
  return o;
}

int resolve_threads(int flag) {
  if (flag > 0) return flag;
  if (const char* env = std::getenv("TSIEVE_THREADS"))
    if (int v = std::atoi(env); v > 0) return v;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? static_cast<int>(hw) : 1;
}

std::vector<int> int_list(const std::string& s, const char* flag) {
  std::vector<int> out;
  std::stringstream ss(s);
  for (std::string tok; std::getline(ss, tok, ',');) {
    if (tok.empty()) continue;
    size_t used = 0;
    int x = 0;
    try {
      x = std::stoi(tok, &used);
    } catch (const std::exception&) {
      used = 0;
    }
    if (used == 0 || used != tok.size())
      throw std::invalid_argument(std::string(flag) + ": malformed integer '" + tok + "'");
    out.push_back(x);
  }
  if (out.empty()) throw std::invalid_argument(std::string(flag) + ": empty list");
  return out;
}

struct Instance {
  LoadResult loaded;
  SolveRequest req;
};

Vertex vertex_named(const LoadResult& lr, const std::string& tok, const char* flag) {
  for (Vertex x = 0; x < static_cast<Vertex>(lr.vertex_names.size()); ++x)
    if (lr.vertex_names[x] == tok) return x;
  throw std::invalid_argument(std::string(flag) + ": unknown vertex '" + tok + "'");
}

Instance load_instance(const Opts& o) {
  Instance inst;
  std::ifstream ef(o.graph_file);
  if (!ef) throw std::invalid_argument("--graph: cannot open " + o.graph_file);
  std::optional<std::ifstream> cf;
  if (!o.colors_file.empty()) {
    cf.emplace(o.colors_file);
    if (!*cf) throw std::invalid_argument("--colors: cannot open " + o.colors_file);
  }
  ef.close();
  inst.loaded = load_graph_file(o.graph_file, cf ? &*cf : nullptr, o.directed, o.ingest_cache);
  if (!o.delays_file.empty()) {
    std::ifstream df(o.delays_file);
    if (!df) throw std::invalid_argument("--delays: cannot open " + o.delays_file);
    inst.loaded.graph.set_delays(load_delays(df, inst.loaded));
  }
  SolveRequest& req = inst.req;
  const auto p = problem_from_name(o.problem);
  if (!p) throw std::invalid_argument("--problem: unknown '" + o.problem + "'");
  req.problem = *p;
  switch (req.problem) {
    case Problem::k_temp_path:
    case Problem::rainbow_path:
    case Problem::sd_colorful_path:
      if (o.k < 1) throw std::invalid_argument("--k must be a positive integer");
      req.query = MotifQuery::size_only(o.k);
      break;
    case Problem::path_motif:
    case Problem::colorful_path: {
      if (o.motif.empty()) throw std::invalid_argument("--motif is required");
      const auto c = int_list(o.motif, "--motif");
      req.query = MotifQuery::from_multiset(std::vector<Color>(c.begin(), c.end()));
      break;
    }
    case Problem::ec_temp_path:
    case Problem::ec_path_motif: {
      if (o.times.empty()) throw std::invalid_argument("--times is required");
      if (req.problem == Problem::ec_path_motif && o.motif.empty())
        throw std::invalid_argument("--motif is required");
      const auto ts = int_list(o.times, "--times");
      std::vector<Color> col;
      if (!o.motif.empty()) {
        const auto c = int_list(o.motif, "--motif");
        col.assign(c.begin(), c.end());
      }
      req.query = MotifQuery::from_times(std::vector<Timestamp>(ts.begin(), ts.end()), col);
      break;
    }
    case Problem::vc_path_motif:
    case Problem::vc_colorful_path: {
      if (o.order.empty()) throw std::invalid_argument("--order is required");
      const auto c = int_list(o.order, "--order");
      req.query = MotifQuery::from_order(std::vector<Color>(c.begin(), c.end()));
      break;
    }
  }
  if (req.problem == Problem::sd_colorful_path) {
    if (o.source.empty() || o.dest.empty())
      throw std::invalid_argument("--source and --dest are required");
    req.source = vertex_named(inst.loaded, o.source, "--source");
    req.dest = vertex_named(inst.loaded, o.dest, "--dest");
  }
  req.wildcard_max = o.wildcards_max;
  if (o.preprocess == "none") req.preprocess = PreprocessLevel::none;
  else if (o.preprocess == "colors") req.preprocess = PreprocessLevel::color_filter;
  else if (o.preprocess == "static") req.preprocess = PreprocessLevel::static_sieve;
  else if (o.preprocess == "both") req.preprocess = PreprocessLevel::both;
  else throw std::invalid_argument("--preprocess: unknown '" + o.preprocess + "'");
  if (o.extraction == "localized") req.extraction = ExtractionStrategy::localized;
  else if (o.extraction == "self-reducible") req.extraction = ExtractionStrategy::self_reducible;
  else throw std::invalid_argument("--extraction: unknown '" + o.extraction + "'");

  SieveConfig& cfg = req.config;
  cfg.seed = o.seed;
  cfg.field_bits = o.field_bits;
  cfg.lane_width = o.lanes;
  cfg.threads = resolve_threads(o.threads);
  tsieve::set_device(o.device);
  // The reference CLI leaves memory_cap_words at its library default (2^31
  // words), which bounds the reference's dense n*W*(t+1) layers.  The
  // engine's working set is O(referenced runs * W) in HBM and the batch width
  // is already fitted to free device memory, so the CLI lifts the cap rather
  // than shrink the batch (a library caller's cap is still honoured).
  cfg.memory_cap_words = std::uint64_t{1} << 62;
  const bool eps = inst.loaded.graph.has_transition_times();
  if (o.edge_model == "auto")
    cfg.edge_model = o.delays_file.empty()
                         ? (eps ? EdgeModel::transition_only : EdgeModel::instant)
                         : (eps ? EdgeModel::transition_delay : EdgeModel::delay_only);
  else if (o.edge_model == "instant") cfg.edge_model = EdgeModel::instant;
  else if (o.edge_model == "transition") cfg.edge_model = EdgeModel::transition_only;
  else if (o.edge_model == "delay") cfg.edge_model = EdgeModel::delay_only;
  else if (o.edge_model == "transition-delay") cfg.edge_model = EdgeModel::transition_delay;
  else throw std::invalid_argument("--edge-model: unknown '" + o.edge_model + "'");
  return inst;
}

const char* model_name(EdgeModel m) {
  switch (m) {
    case EdgeModel::instant: return "instant";
    case EdgeModel::transition_only: return "transition";
    case EdgeModel::delay_only: return "delay";
    case EdgeModel::transition_delay: return "transition-delay";
  }
  return "?";
}

Json record(const std::string& command, const Opts& o, const Instance& inst,
            const SolveReport& r) {
  const TemporalGraph& g = inst.loaded.graph;
  const SieveConfig& c = inst.req.config;
  char cs[32];
  std::snprintf(cs, sizeof cs, "%016llx", static_cast<unsigned long long>(r.checksum));
  Json::Arr flagged;
  for (Vertex x : r.flagged) flagged.push_back(x);
  Json::Obj j{
      {"command", command},
      {"problem", problem_name(inst.req.problem)},
      {"graph", Json::Obj{{"n", g.n()}, {"m", g.m()}, {"t", g.t()}, {"directed", g.directed()}}},
      {"config", Json::Obj{{"seed", c.seed},
                           {"field_bits", c.field_bits},
                           {"lanes", c.lane_width},
                           {"threads", c.threads},
                           {"preprocess", o.preprocess},
                           {"extraction", o.extraction},
                           {"edge_model", model_name(c.edge_model)}}},
      {"decision", r.decision ? "YES" : "NO"},
      {"certain", r.certain},
      {"flagged", flagged},
      {"fn_bound", r.fn_bound},
      {"oracle_calls", r.oracle_calls},
      {"timings", Json::Obj{{"preprocess_s", r.timings.preprocess_s},
                            {"sieve_s", r.timings.sieve_s},
                            {"extract_s", r.timings.extract_s}}},
      {"peak_field_words", r.peak_field_words},
      {"peak_bytes", r.peak_field_words * static_cast<std::uint64_t>(c.field_bits / 8)},
      {"accumulator_checksum", cs},
      {"preprocessed", Json::Obj{{"n", r.preprocessed_n}, {"m", r.preprocessed_m}}},
      {"wildcards_used", r.wildcards_used},
      {"note", r.note},
      {"engine", "b200"},
  };
  j["optimum_ts"] = r.optimum_ts >= 0 ? Json(r.optimum_ts) : Json(nullptr);
  if (r.witness) {
    Json::Arr verts, names, edges;
    for (Vertex x : r.witness->vertices) {
      verts.push_back(x);
      names.push_back(inst.loaded.vertex_names[x]);
    }
    for (const TemporalEdge& e : r.witness->edges) edges.push_back(Json::Arr{e.u, e.v, e.ts});
    j["witness"] = Json::Obj{{"vertices", verts}, {"vertex_names", names}, {"edges", edges}};
  } else {
    j["witness"] = nullptr;
  }
  j["extraction_failed"] = r.extraction_failed;
  return j;
}

void print_text(const Json& j) {
  auto s = [&](const Json* x) -> std::string {
    if (!x) return "";
    std::ostringstream os;
    if (auto* str = std::get_if<std::string>(&x->v)) return *str;
    dump(os, *x, 0);
    return os.str();
  };
  const Json& g = *j.get("graph");
  const Json& c = *j.get("config");
  std::cout << "problem:    " << s(j.get("problem")) << "\n"
            << "graph:      n=" << s(g.get("n")) << " m=" << s(g.get("m")) << " t=" << s(g.get("t"))
            << "\n"
            << "config:     seed=" << s(c.get("seed")) << " b=" << s(c.get("field_bits"))
            << " W=" << s(c.get("lanes")) << " threads=" << s(c.get("threads"))
            << " preprocess=" << s(c.get("preprocess")) << "\n"
            << "decision:   " << s(j.get("decision"))
            << (std::get<bool>(j.get("certain")->v) ? " (exact)" : "") << "\n";
  if (!j.get("optimum_ts")->is_null()) std::cout << "optimum-ts: " << s(j.get("optimum_ts")) << "\n";
  if (const Json* w = j.get("witness"); !w->is_null()) {
    std::cout << "witness:   ";
    for (const Json& e : w->get("edges")->as_arr()) {
      const auto& a = e.as_arr();
      std::cout << " (" << a[0].as_int() << "," << a[1].as_int() << "@" << a[2].as_int() << ")";
    }
    std::cout << "\n";
  }
  if (std::get<bool>(j.get("extraction_failed")->v)) std::cout << "extraction: FAILED\n";
  std::cout << "flagged:    " << j.get("flagged")->as_arr().size() << " vertices\n"
            << "fn-bound:   " << s(j.get("fn_bound")) << "\n"
            << "timings:    preprocess=" << s(j.get("timings")->get("preprocess_s"))
            << "s sieve=" << s(j.get("timings")->get("sieve_s"))
            << "s extract=" << s(j.get("timings")->get("extract_s")) << "s\n"
            << "peak-mem:   " << s(j.get("peak_field_words")) << " field words ("
            << s(j.get("peak_bytes")) << " bytes)\n"
            << "checksum:   " << s(j.get("accumulator_checksum")) << "\n";
  if (!s(j.get("note")).empty()) std::cout << "note:       " << s(j.get("note")) << "\n";
}

int run_solver(const std::string& command, const Opts& o, SolveMode mode) {
  Instance inst = load_instance(o);
  if (mode == SolveMode::extract && o.optimize) mode = SolveMode::extract_optimum;
  const SolveReport r = solve(inst.loaded.graph, inst.loaded.coloring, inst.req, mode);
  const Json j = record(command, o, inst, r);
  if (o.format == "json") {
    dump(std::cout, j, 0);
    std::cout << "\n";
  } else {
    print_text(j);
  }
  const bool wanted = mode == SolveMode::extract || mode == SolveMode::extract_optimum;
  if (r.decision && wanted && r.extraction_failed) return kBudget;
  return r.decision ? kYes : kNo;
}

int run_verify(const Opts& o) {
  Instance inst = load_instance(o);
  std::ifstream wf(o.witness_file);
  if (!wf) throw std::invalid_argument("--witness: cannot open " + o.witness_file);
  std::stringstream ss;
  ss << wf.rdbuf();
  const Json doc = Reader(ss.str()).parse();
  const Json* w = doc.get("witness");
  if (!w || w->is_null()) w = &doc;
  if (!w->get("vertices") || !w->get("edges"))
    throw std::invalid_argument("witness file lacks vertices/edges");
  TemporalPath p;
  for (const Json& x : w->get("vertices")->as_arr()) p.vertices.push_back(static_cast<Vertex>(x.as_int()));
  for (const Json& e : w->get("edges")->as_arr()) {
    const auto& a = e.as_arr();
    if (a.size() < 3) throw std::invalid_argument("witness edge needs [u, v, ts]");
    p.edges.push_back({static_cast<Vertex>(a[0].as_int()), static_cast<Vertex>(a[1].as_int()),
                       static_cast<Timestamp>(a[2].as_int()), 1});
  }
  const EffectiveInstance eff =
      effective_instance(inst.loaded.graph, inst.loaded.coloring, inst.req);
  const PathVerdict v = validate_path(inst.loaded.graph, eff.coloring, p, eff.query,
                                      inst.req.config.edge_model, eff.anchor.source,
                                      eff.anchor.sink);
  if (v) {
    std::cout << "witness OK\n";
    return kYes;
  }
  std::cout << "witness INVALID: " << v.detail << "\n";
  return kNo;
}

void usage(std::ostream& os) {
  os << "color-constrained temporal path detection and extraction (B200 engine)\n"
        "usage: tsieve <decide|extract|optimum|verify> --graph FILE [options]\n"
        "  --colors FILE --problem NAME --motif C,C,.. --k K --source S --dest D\n"
        "  --seed N --field-bits 64 --lanes W --threads T --preprocess none|colors\n"
        "  --extraction localized|self-reducible --edge-model auto|instant\n"
        "  --wildcards-max K --directed --format text|json --device D\n"
        "  extract: --optimize/--no-optimize   verify: --witness FILE\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    std::cerr << "A subcommand is required\n";
    return kUsage;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage(std::cout);
    return kYes;
  }
  try {
    if (cmd != "decide" && cmd != "extract" && cmd != "optimum" && cmd != "verify")
      throw UsageError("unknown subcommand '" + cmd + "'");
    const Opts o = parse_flags(cmd, argc - 2, argv + 2);
    if (cmd == "decide") return run_solver(cmd, o, SolveMode::decide);
    if (cmd == "extract") return run_solver(cmd, o, SolveMode::extract);
    if (cmd == "optimum") return run_solver(cmd, o, SolveMode::optimum);
    return run_verify(o);
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return kUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  }
}
