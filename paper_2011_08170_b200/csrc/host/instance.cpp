// instance.cpp — instance format and host-side text I/O (out of the GPU path by design:
// SURVEY.md §2 rows 2 and 8). TSPLIB EUC_2D subset with the reference's acceptance rules
// (instance.cpp:39-98 there), %.17g round-trip serialization, synthetic generators, CPLEX-LP
// export, benchmark rows. Scalar accessors (distance) mirror instance.cpp:126-141.
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <istream>
#include <map>
#include <ostream>
#include <sstream>

#include "f2m/api.hpp"

namespace f2m {
inline namespace b200 {

namespace {

std::string strip(const std::string& s) {
  const char* ws = " \t\r\n";
  const size_t a = s.find_first_not_of(ws);
  if (a == std::string::npos) return {};
  return s.substr(a, s.find_last_not_of(ws) - a + 1);
}

std::string to_upper(std::string s) {
  for (char& c : s) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
  return s;
}

}  // namespace

Instance parse_tsplib(std::istream& in) {
  Instance inst;
  long dim = -1;
  bool have_coords = false;
  std::string raw;
  while (std::getline(in, raw)) {
    const std::string line = strip(raw);
    if (line.empty()) continue;
    const size_t colon = line.find(':');
    const std::string key = to_upper(strip(colon == std::string::npos ? line : line.substr(0, colon)));
    const std::string val = colon == std::string::npos ? std::string() : strip(line.substr(colon + 1));
    if (key == "EOF") break;
    if (key == "NAME") {
      inst.name = val;
    } else if (key == "DIMENSION") {
      try {
        dim = std::stoi(val);
      } catch (const std::exception&) {
        throw ParseError("DIMENSION is not an integer: '" + val + "'");
      }
      if (dim < 1) throw ParseError("DIMENSION must be positive");
    } else if (key == "EDGE_WEIGHT_TYPE") {
      if (to_upper(val) != "EUC_2D") throw ParseError("unsupported EDGE_WEIGHT_TYPE '" + val + "' (only EUC_2D)");
    } else if (key == "NODE_COORD_SECTION") {
      if (dim < 1) throw ParseError("NODE_COORD_SECTION before DIMENSION");
      inst.points.assign(static_cast<size_t>(dim), Point{});
      std::vector<char> seen(static_cast<size_t>(dim), 0);
      for (long row = 0; row < dim; ++row) {
        long long id = 0;
        double x = 0.0, y = 0.0;
        if (!(in >> id >> x >> y))
          throw ParseError("bad or missing coordinate line " + std::to_string(row + 1) + " of " + std::to_string(dim));
        if (id < 1 || id > dim)
          throw ParseError("node index " + std::to_string(id) + " out of range 1.." + std::to_string(dim));
        if (!std::isfinite(x) || !std::isfinite(y))
          throw ParseError("non-finite coordinate at node " + std::to_string(id));
        if (seen[static_cast<size_t>(id - 1)]) throw ParseError("duplicate node index " + std::to_string(id));
        seen[static_cast<size_t>(id - 1)] = 1;
        inst.points[static_cast<size_t>(id - 1)] = Point{x, y};
      }
      std::getline(in, raw);  // remainder of the last coordinate line
      have_coords = true;
    }
    // other keywords (TYPE, COMMENT, ...) are ignored
  }
  if (dim < 1) throw ParseError("missing DIMENSION");
  if (!have_coords) throw ParseError("missing NODE_COORD_SECTION");
  inst.mode = DistanceMode::kEuc2dRounded;  // TSPLIB EUC_2D is nearest-integer
  return inst;
}

Instance parse_tsplib_string(const std::string& text) {
  std::istringstream in(text);
  return parse_tsplib(in);
}

Instance load_tsplib_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open '" + path + "'");
  return parse_tsplib(in);
}

void serialize_tsplib(const Instance& instance, std::ostream& out) {
  out << "NAME : " << instance.name << "\nTYPE : TSP\nDIMENSION : " << instance.node_count()
      << "\nEDGE_WEIGHT_TYPE : EUC_2D\nNODE_COORD_SECTION\n";
  char line[96];
  for (int i = 0; i < instance.node_count(); ++i) {
    std::snprintf(line, sizeof(line), "%d %.17g %.17g\n", i + 1, instance.points[i].x, instance.points[i].y);
    out << line;
  }
  out << "EOF\n";
}

double distance(const Instance& instance, int i, int j) {
  const int n = instance.node_count();
  if (i < 0 || j < 0 || i >= n || j >= n)
    throw IndexError("node index out of range: (" + std::to_string(i) + ", " + std::to_string(j) +
                     ") with n=" + std::to_string(n));
  const double dx = instance.points[i].x - instance.points[j].x;
  const double dy = instance.points[i].y - instance.points[j].y;
  const double d = std::sqrt(dx * dx + dy * dy);
  return instance.mode == DistanceMode::kEuc2dRounded ? std::floor(d + 0.5) : d;
}

Instance generate_instance(int n, std::uint64_t seed, double box) {
  if (n < 1) throw ArgumentError("generate_instance: n must be >= 1");
  if (!(box > 0.0)) throw ArgumentError("generate_instance: box must be > 0");
  Instance inst;
  inst.name = "rand" + std::to_string(n) + "-s" + std::to_string(seed);
  inst.mode = DistanceMode::kEuc2dExact;
  inst.points.resize(static_cast<size_t>(n));
  SplitMix64 rng(seed);
  for (auto& p : inst.points) {  // x then y per point
    p.x = rng.next_double() * box;
    p.y = rng.next_double() * box;
  }
  return inst;
}

Instance generate_clustered_instance(int n, std::uint64_t seed, double box) {
  if (n < 1) throw ArgumentError("generate_clustered_instance: n must be >= 1");
  if (!(box > 0.0)) throw ArgumentError("generate_clustered_instance: box must be > 0");
  Instance inst;
  inst.name = "clust" + std::to_string(n) + "-s" + std::to_string(seed);
  inst.mode = DistanceMode::kEuc2dExact;
  SplitMix64 rng(seed);
  const int centres = std::max(1, n / 10);
  std::vector<Point> c(static_cast<size_t>(centres));
  for (auto& p : c) {
    p.x = rng.next_double() * box;
    p.y = rng.next_double() * box;
  }
  const double sigma = box / std::sqrt(static_cast<double>(n));
  const double two_pi = 6.283185307179586476925286766559;
  inst.points.resize(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const double u1 = rng.next_double(), u2 = rng.next_double();
    const double r = std::sqrt(-2.0 * std::log(1.0 - u1));  // 1 - u1 in (0, 1]
    const Point& ctr = c[static_cast<size_t>(i % centres)];
    inst.points[i].x = ctr.x + sigma * r * std::cos(two_pi * u2);
    inst.points[i].y = ctr.y + sigma * r * std::sin(two_pi * u2);
  }
  return inst;
}

// ------------------------------------------------------------------ LP export

void write_lp(const Graph& graph, std::ostream& out) {
  if (graph.edge_count() == 0) throw ArgumentError("write_lp: empty graph");
  const auto& edges = graph.edges();
  auto name = [&](int e) { return "x_" + std::to_string(edges[e].u) + "_" + std::to_string(edges[e].v); };
  char num[64];
  out << "Minimize\n obj:";
  for (int e = 0; e < graph.edge_count(); ++e) {
    std::snprintf(num, sizeof(num), "%.17g", edges[e].cost);
    out << (e == 0 ? " " : " + ") << num << ' ' << name(e);
  }
  out << "\nSubject To\n";
  for (int v = 0; v < graph.node_count(); ++v) {
    out << " deg_" << v << ":";
    const auto inc = graph.incident(v);
    for (size_t i = 0; i < inc.size(); ++i) out << (i == 0 ? " " : " + ") << name(inc[i]);
    out << " = 2\n";
  }
  out << "Bounds\n";
  for (int e = 0; e < graph.edge_count(); ++e) out << " 0 <= " << name(e) << " <= 1\n";
  out << "End\n";
}

// ------------------------------------------------------------------ benchmark rows

InstanceSource InstanceSource::from_file(std::string p) {
  InstanceSource s;
  s.path = std::move(p);
  return s;
}

InstanceSource InstanceSource::synthetic(int n, std::uint64_t seed, double box) {
  InstanceSource s;
  s.synthetic_n = n;
  s.seed = seed;
  s.box = box;
  return s;
}

Instance InstanceSource::load() const {
  return path.empty() ? generate_instance(synthetic_n, seed, box) : load_tsplib_file(path);
}

std::string InstanceSource::id() const {
  if (path.empty()) return "rand" + std::to_string(synthetic_n) + "-s" + std::to_string(seed);
  std::string base = path.substr(path.find_last_of("/\\") == std::string::npos ? 0 : path.find_last_of("/\\") + 1);
  const size_t dot = base.find_last_of('.');
  return dot == std::string::npos ? base : base.substr(0, dot);
}

std::vector<BenchRow> run_benchmark(const std::vector<InstanceSource>& sources, const RunConfig& config) {
  std::vector<BenchRow> rows;
  for (const InstanceSource& src : sources) {
    BenchRow row;
    row.instance = src.id();
    const auto t0 = std::chrono::steady_clock::now();
    try {
      const Instance inst = src.load();
      row.nodes = inst.node_count();
      const Graph g = build_knn_graph(inst, std::max(3, std::min(config.k, inst.node_count() - 1)));
      row.edges = g.edge_count();
      const SolveOutcome o = full_solve_graph(g, config);
      row.sweeps = o.convergence.sweeps;
      row.gap = o.verification.duality_gap;
      row.restarts = o.restarts;
      row.ok = true;
    } catch (const std::exception& e) {
      row.ok = false;
      row.error = e.what();
      row.gap = std::nan("");
    }
    row.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rows.push_back(std::move(row));
  }
  return rows;
}

void write_bench_csv(const std::vector<BenchRow>& rows, std::ostream& out) {
  out << "instance,nodes,edges,sweeps,seconds,gap,restarts\n";
  char line[256];
  for (const BenchRow& r : rows) {
    std::snprintf(line, sizeof(line), "%s,%d,%d,%d,%.6f,%.12g,%d\n", r.instance.c_str(), r.nodes, r.edges,
                  r.sweeps, r.seconds, r.gap, r.restarts);
    out << line;
  }
}

static std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (const char c : s) {
    if (c == '"' || c == '\\') { o += '\\'; o += c; }
    else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof(b), "\\u%04x", static_cast<unsigned char>(c));
      o += b;
    } else o += c;
  }
  return o + "\"";
}

static std::string json_number(double v) {
  if (std::isnan(v)) return "null";
  char b[64];
  for (int prec = 15; prec <= 17; ++prec) {  // shortest representation that round-trips
    std::snprintf(b, sizeof(b), "%.*g", prec, v);
    if (std::strtod(b, nullptr) == v) break;
  }
  std::string s = b;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

void write_bench_json(const std::vector<BenchRow>& rows, std::ostream& out) {
  // keys in lexicographic order, 2-space indent (the reference's nlohmann::json dump(2) layout)
  out << "[";
  for (size_t i = 0; i < rows.size(); ++i) {
    const BenchRow& r = rows[i];
    std::map<std::string, std::string> kv;
    kv["instance"] = json_string(r.instance);
    kv["nodes"] = std::to_string(r.nodes);
    kv["edges"] = std::to_string(r.edges);
    kv["sweeps"] = std::to_string(r.sweeps);
    kv["seconds"] = json_number(r.seconds);
    kv["restarts"] = std::to_string(r.restarts);
    kv["ok"] = r.ok ? "true" : "false";
    kv["gap"] = json_number(r.gap);
    if (!r.error.empty()) kv["error"] = json_string(r.error);
    out << (i == 0 ? "\n" : ",\n") << "  {";
    size_t j = 0;
    for (const auto& [k, v] : kv) out << (j++ == 0 ? "\n" : ",\n") << "    " << json_string(k) << ": " << v;
    out << "\n  }";
  }
  out << (rows.empty() ? "]" : "\n]") << "\n";
}

}  // namespace b200
}  // namespace f2m
