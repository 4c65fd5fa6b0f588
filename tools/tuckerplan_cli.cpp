// tuckerplan command line on the B200 engine: plan, simulate, gen-tensor, hooi.
//
// Same subcommands, flags, output text, file formats and exit codes as the reference's tool
// (tools/tuckerplan_cli.cpp:1-563, README.md "Command line") for the commands that touch the engine and its plans;
// `bench` (corpus statistics of bench.hpp) is not provided.  Written against include/tuckerplan/*.hpp, i.e. the
// calls below are the reference's API; `hooi` keeps the tensor resident on the GPU between sweeps (DeviceHooi).
//
// Exit codes: 0 success, 1 invalid input or infeasible request, 2 traced simulation disagreed with the volume model
// on a TTM count.
#include <cstdio>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <memory>
#include <string>
#include <vector>

#include "tuckerplan/serialize.hpp"
#include "tuckerplan/tuckerplan.hpp"

namespace tp = tuckerplan;
using tp::u64;

namespace {

// ---- arguments ---------------------------------------------------------------------------------------------
struct OptionSpec {
  const char* name;
  bool flag;
  const char* help;
};

struct Command {
  const char* name;
  const char* summary;
  std::vector<OptionSpec> options;
};

const std::vector<Command>& commands() {
  static const std::vector<Command> all = {
      {"plan", "choose a tree and grids for a spec",
       {{"--spec", false, "spec JSON file {\"L\":[...],\"K\":[...]}"},
        {"--L", false, "mode lengths, comma separated"},
        {"--K", false, "core lengths, comma separated"},
        {"--procs", false, "processor count (default 1)"},
        {"--tree", false, "chain-input|chain-k|chain-h|balanced|opt (default opt)"},
        {"--grid", false, "scheme simulate replays: static|dynamic (default dynamic)"},
        {"--legacy-regrid", true, "pick regrid targets by child sum alone"},
        {"--out", false, "write the plan JSON here"},
        {"--format", false, "stdout format: text|json (default text)"}}},
      {"simulate", "replay a plan over block layouts",
       {{"--plan", false, "plan JSON from the plan command"},
        {"--spec", false, "spec JSON file (instead of --plan)"},
        {"--L", false, "mode lengths, comma separated"},
        {"--K", false, "core lengths, comma separated"},
        {"--procs", false, "processor count (default 1)"},
        {"--tree", false, "tree strategy when not using --plan (default opt)"},
        {"--grid", false, "override: static|dynamic"},
        {"--trace", true, "count every element; exits 2 on TTM mismatch"},
        {"--out", false, "write the ledger JSON here"},
        {"--format", false, "stdout format: text|json (default text)"}}},
      {"gen-tensor", "write a seeded random tensor",
       {{"--L", false, "mode lengths, comma separated (required)"},
        {"--seed", false, "generator seed (default 0)"},
        {"--out", false, "output path (required)"}}},
      {"hooi", "run alternating sweeps on dense data (B200)",
       {{"--tensor", false, "tensor file from gen-tensor"},
        {"--L", false, "generate the input instead: lengths"},
        {"--K", false, "core lengths, comma separated (required)"},
        {"--seed", false, "seed for the input and the starting factors (default 0)"},
        {"--tree", false, "tree strategy (default fits the scheme)"},
        {"--scheme", false, "jacobi|gauss-seidel (default gauss-seidel)"},
        {"--sweeps", false, "sweep count (default 5)"},
        {"--init", false, "starting factors: random (default, as the reference) or sthosvd"},
        {"--procs", false, "run on a processor grid of this many GPUs (jacobi only; default 1)"},
        {"--grid", false, "grid for --procs, e.g. 1x1x8 (default: the volume-optimal static grid)"},
        {"--dynamic", true, "with --procs: per-node grids (optimal_dynamic_scheme) instead of one static grid"},
        {"--out", false, "write the sweep report JSON here"},
        {"--format", false, "stdout format: text|json (default text)"}}},
  };
  return all;
}

void print_usage(const Command* cmd) {
  if (!cmd) {
    std::puts("planning and HOOI sweeps for dense Tucker mode products (B200 engine)\n\nsubcommands:");
    for (const Command& c : commands()) std::printf("  %-11s %s\n", c.name, c.summary);
    std::puts("\n`<subcommand> --help` lists its flags.");
    return;
  }
  std::printf("%s: %s\n", cmd->name, cmd->summary);
  for (const OptionSpec& o : cmd->options) std::printf("  %-16s %s\n", o.name, o.help);
}

struct Args {
  std::map<std::string, std::string> values;
  std::set<std::string> flags;
  std::string get(const char* name, const char* fallback = "") const {
    const auto it = values.find(name);
    return it == values.end() ? std::string(fallback) : it->second;
  }
  bool has(const char* name) const { return values.count(name) != 0; }
  bool flag(const char* name) const { return flags.count(name) != 0; }
};

u64 parse_u64(const std::string& item, const std::string& what) {
  std::size_t pos = 0;
  u64 v = 0;
  try {
    if (item.empty() || item[0] == '-' || item[0] == '+') throw std::invalid_argument(item);
    v = std::stoull(item, &pos);
  } catch (const std::exception&) {
    tp::fail(tp::Errc::bad_argument, what + ": bad number " + item);
  }
  if (pos != item.size()) tp::fail(tp::Errc::bad_argument, what + ": bad number " + item);
  return v;
}

std::vector<u64> parse_u64_list(const std::string& text, const char* what) {
  std::vector<u64> values;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) {
    if (item.empty()) continue;
    values.push_back(parse_u64(item, what));
  }
  if (values.empty()) tp::fail(tp::Errc::bad_argument, std::string(what) + ": empty list");
  return values;
}

tp::TreeStrategy strategy_from_name(const std::string& name) {
  for (tp::TreeStrategy st : {tp::TreeStrategy::chain_input, tp::TreeStrategy::chain_by_cost,
                              tp::TreeStrategy::chain_by_ratio, tp::TreeStrategy::balanced, tp::TreeStrategy::optimal})
    if (name == tp::strategy_name(st)) return st;
  tp::fail(tp::Errc::bad_argument, "unknown tree strategy: " + name);
}

tp::json load_json_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) tp::fail(tp::Errc::bad_argument, "cannot open " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  const tp::json j = tp::json::parse(ss.str());
  if (j.is_discarded()) tp::fail(tp::Errc::bad_argument, "bad JSON in " + path);
  return j;
}

void write_text_file(const std::string& path, const std::string& content) {
  std::ofstream out(path);
  if (!out) tp::fail(tp::Errc::bad_argument, "cannot open " + path);
  out << content;
  if (!out) tp::fail(tp::Errc::bad_argument, "write failed: " + path);
}

std::string join(const std::vector<u64>& v, const char* sep) {
  std::string s;
  for (std::size_t i = 0; i < v.size(); ++i) s += (i ? sep : "") + std::to_string(v[i]);
  return s;
}

std::string spec_id(const tp::ProblemSpec& s) { return "L" + join(s.L, "x") + "-K" + join(s.K, "x"); }  // bench.hpp:222-230

std::string node_label(const tp::TtmTree& t, int id) {
  const tp::TreeNode& n = t.nodes[id];
  if (n.kind == tp::NodeKind::root) return "T";
  return (n.kind == tp::NodeKind::mode ? "M" : "F") + std::to_string(n.mode + 1);
}

// spec from --spec file or inline --L/--K; exactly one source
tp::ProblemSpec resolve_spec(const Args& a) {
  const bool inline_given = a.has("--L") || a.has("--K");
  if (a.has("--spec") && inline_given) tp::fail(tp::Errc::bad_argument, "give either --spec or --L/--K, not both");
  if (a.has("--spec")) return tp::spec_from_json(load_json_file(a.get("--spec")));
  if (!a.has("--L") || !a.has("--K")) tp::fail(tp::Errc::bad_argument, "need --spec or both --L and --K");
  tp::ProblemSpec s;
  s.L = parse_u64_list(a.get("--L"), "--L");
  s.K = parse_u64_list(a.get("--K"), "--K");
  tp::validate_spec(s);
  return s;
}

// ---- plans (tools/tuckerplan_cli.cpp:105-215) ------------------------------------------------------------------
struct Plan {
  tp::ProblemSpec spec;
  std::string strategy;
  tp::TtmTree tree;
  u64 procs = 1;
  std::string grid_kind;  // "static" or "dynamic": which scheme simulate replays
  tp::CostReport cost;
  tp::Grid static_grid;
  tp::VolumeReport static_volume;
  tp::DynamicGridScheme dynamic_scheme;
  tp::VolumeReport dynamic_volume;
};

Plan make_plan(const tp::ProblemSpec& spec, const std::string& strategy, u64 procs, const std::string& grid_kind,
               bool legacy_regrid) {
  if (procs < 1) tp::fail(tp::Errc::bad_argument, "--procs must be at least 1");
  if (grid_kind != "static" && grid_kind != "dynamic") tp::fail(tp::Errc::bad_argument, "--grid must be static or dynamic");
  Plan p;
  p.spec = spec;
  p.strategy = strategy;
  // through the label form, so node ids match a reloaded plan
  p.tree = tp::tree_from_json(tp::tree_to_json(tp::build_tree(spec, strategy_from_name(strategy))));
  tp::validate_tree(p.tree, spec);
  p.procs = procs;
  p.grid_kind = grid_kind;
  p.cost = tp::tree_cost(p.tree, spec);
  const tp::StaticGridResult st = tp::optimal_static_grid(p.tree, spec, procs);
  p.static_grid = st.grid;
  p.static_volume = st.report;
  tp::DynamicOptions opts;
  opts.legacy_regrid_target = legacy_regrid;
  const tp::DynamicSchemeResult dyn = tp::optimal_dynamic_scheme(p.tree, spec, procs, opts);
  p.dynamic_scheme = dyn.scheme;
  p.dynamic_volume = dyn.report;
  return p;
}

tp::json plan_to_json(const Plan& p) {
  return tp::json::object({{"format", tp::json("tuckerplan-plan-v1")},
                           {"spec", tp::spec_to_json(p.spec)},
                           {"strategy", tp::json(p.strategy)},
                           {"procs", tp::json(p.procs)},
                           {"grid", tp::json(p.grid_kind)},
                           {"tree", tp::tree_to_json(p.tree)},
                           {"cost", tp::cost_to_json(p.cost)},
                           {"static_grid", tp::grid_to_json(p.static_grid)},
                           {"static_volume", tp::volume_to_json(p.static_volume)},
                           {"dynamic_scheme", tp::scheme_to_json(p.dynamic_scheme)},
                           {"dynamic_volume", tp::volume_to_json(p.dynamic_volume)}});
}

Plan plan_from_json(const tp::json& j) {
  for (const char* key : {"spec", "procs", "grid", "tree", "static_grid", "dynamic_scheme"})
    if (!j.is_object() || !j.contains(key)) tp::fail(tp::Errc::bad_argument, std::string("plan file lacks ") + key);
  Plan p;
  p.spec = tp::spec_from_json(j.at("spec"));
  p.strategy = j.contains("strategy") ? j.at("strategy").as_string() : std::string("custom");
  p.tree = tp::tree_from_json(j.at("tree"));
  tp::validate_tree(p.tree, p.spec);
  p.procs = j.at("procs").as_u64();
  p.grid_kind = j.at("grid").as_string();
  p.cost = tp::tree_cost(p.tree, p.spec);
  p.static_grid = tp::grid_from_json(j.at("static_grid"));
  p.static_volume = tp::static_volume(p.tree, p.spec, p.static_grid, p.procs);
  p.dynamic_scheme = tp::scheme_from_json(j.at("dynamic_scheme"));
  p.dynamic_volume = tp::scheme_volume(p.tree, p.spec, p.dynamic_scheme, p.procs);
  return p;
}

std::string plan_to_text(const Plan& p) {
  std::string out;
  out += "spec      " + spec_id(p.spec) + "\n";
  out += "tree      " + p.strategy + ": " + std::to_string(p.cost.total_macs) + " MACs over " +
         std::to_string(p.cost.n_internal) + " nodes, depth " + std::to_string(p.cost.depth) + "\n";
  out += "procs     " + std::to_string(p.procs) + "\n";
  out += "static    grid " + join(p.static_grid.q, "x") + ", volume " + std::to_string(p.static_volume.total) + "\n";
  out += "dynamic   volume " + std::to_string(p.dynamic_volume.total) + ", root grid " +
         join(p.dynamic_scheme.root.q, "x") + "\n";
  for (const tp::NodeVolume& nv : p.dynamic_volume.per_node)
    if (nv.regrid)
      out += "          node " + std::to_string(nv.node) + " [" + node_label(p.tree, nv.node) + "] regrids to " +
             join(p.dynamic_scheme.node_grids.at(nv.node).q, "x") + "\n";
  out += "selected  " + p.grid_kind + "\n";
  return out;
}

std::string ledger_to_text(const Plan& p, const tp::SimLedger& led) {
  std::string out;
  for (const tp::NodeTrace& nt : led.nodes) {
    out += "node " + std::to_string(nt.node) + " [" + node_label(p.tree, nt.node) + "]: flops " +
           std::to_string(nt.flops) + ", ttm " + std::to_string(nt.model_ttm) + ", regrid " +
           std::to_string(nt.model_regrid);
    if (led.traced)
      out += " (measured ttm " + std::to_string(nt.measured_ttm) + ", regrid " + std::to_string(nt.measured_regrid) + ")";
    out += "\n";
  }
  out += "totals: flops " + std::to_string(led.total_flops) + ", ttm " + std::to_string(led.total_model_ttm) +
         ", regrid " + std::to_string(led.total_model_regrid);
  if (led.traced)
    out += " (measured ttm " + std::to_string(led.total_measured_ttm) + ", regrid " +
           std::to_string(led.total_measured_regrid) + ")";
  out += ", peak live " + std::to_string(led.peak_live) + "\n";
  return out;
}

void check_format(const std::string& format) {
  if (format != "text" && format != "json") tp::fail(tp::Errc::bad_argument, "--format must be text or json");
}

void emit(const std::string& json_body, const std::string& text_body, const Args& a) {
  const std::string format = a.get("--format", "text");
  check_format(format);
  if (a.has("--out")) write_text_file(a.get("--out"), json_body);
  std::fputs(format == "json" ? json_body.c_str() : text_body.c_str(), stdout);
}

int cmd_plan(const Args& a) {
  const tp::ProblemSpec spec = resolve_spec(a);
  const Plan plan = make_plan(spec, a.get("--tree", "opt"), a.has("--procs") ? parse_u64(a.get("--procs"), "--procs") : 1,
                              a.get("--grid", "dynamic"), a.flag("--legacy-regrid"));
  emit(plan_to_json(plan).dump(2) + "\n", plan_to_text(plan), a);
  return 0;
}

int cmd_simulate(const Args& a) {
  Plan p;
  std::string kind;
  if (a.has("--plan")) {
    if (a.has("--spec") || a.has("--L") || a.has("--K"))
      tp::fail(tp::Errc::bad_argument, "give either --plan or a spec, not both");
    p = plan_from_json(load_json_file(a.get("--plan")));
    kind = a.has("--grid") ? a.get("--grid") : p.grid_kind;
  } else {
    p = make_plan(resolve_spec(a), a.get("--tree", "opt"), a.has("--procs") ? parse_u64(a.get("--procs"), "--procs") : 1,
                  a.get("--grid", "dynamic"), false);
    kind = p.grid_kind;
  }
  tp::DynamicGridScheme scheme;
  if (kind == "static")
    scheme = tp::uniform_scheme(p.tree, p.static_grid);
  else if (kind == "dynamic")
    scheme = p.dynamic_scheme;
  else
    tp::fail(tp::Errc::bad_argument, "--grid must be static or dynamic");
  const tp::SimLedger led = tp::simulate_distribution(p.tree, p.spec, scheme, p.procs, a.flag("--trace"));
  emit(tp::ledger_to_json(led).dump(2) + "\n", ledger_to_text(p, led), a);
  if (led.traced)
    for (const tp::NodeTrace& nt : led.nodes)
      if (nt.measured_ttm != nt.model_ttm) {
        std::fprintf(stderr, "model violation: node %d measured ttm %llu != model %llu\n", nt.node,
                     static_cast<unsigned long long>(nt.measured_ttm), static_cast<unsigned long long>(nt.model_ttm));
        return 2;
      }
  return 0;
}

int cmd_gen_tensor(const Args& a) {
  if (!a.has("--L") || !a.has("--out")) tp::fail(tp::Errc::bad_argument, "gen-tensor needs --L and --out");
  const std::vector<u64> lens = parse_u64_list(a.get("--L"), "--L");
  const u64 seed = a.has("--seed") ? parse_u64(a.get("--seed"), "--seed") : 0;
  const tp::DenseTensor t = tp::random_tensor(std::vector<std::size_t>(lens.begin(), lens.end()), seed);
  tp::write_tensor(a.get("--out"), t);
  std::printf("wrote %s: dims %s, %zu elements\n", a.get("--out").c_str(), join(lens, "x").c_str(), t.size());
  return 0;
}

int cmd_hooi(const Args& a) {
  if (!a.has("--K")) tp::fail(tp::Errc::bad_argument, "hooi needs --K");
  if (a.has("--tensor") == a.has("--L")) tp::fail(tp::Errc::bad_argument, "need exactly one of --tensor or --L");
  check_format(a.get("--format", "text"));
  const u64 seed = a.has("--seed") ? parse_u64(a.get("--seed"), "--seed") : 0;
  const u64 sweeps = a.has("--sweeps") ? parse_u64(a.get("--sweeps"), "--sweeps") : 5;
  tp::DenseTensor t;
  if (a.has("--tensor")) {
    t = tp::read_tensor(a.get("--tensor"));
  } else {
    const std::vector<u64> lens = parse_u64_list(a.get("--L"), "--L");
    t = tp::random_tensor(std::vector<std::size_t>(lens.begin(), lens.end()), seed);
  }
  tp::ProblemSpec s;
  for (std::size_t d : t.dims) s.L.push_back(d);
  s.K = parse_u64_list(a.get("--K"), "--K");
  tp::validate_spec(s);

  const std::string scheme_name = a.get("--scheme", "gauss-seidel");
  tp::SweepKind kind;
  std::string tree_choice = a.get("--tree");
  if (scheme_name == "jacobi") {
    kind = tp::SweepKind::jacobi;
    if (tree_choice.empty()) tree_choice = "opt";
  } else if (scheme_name == "gauss-seidel") {
    kind = tp::SweepKind::gauss_seidel;
    if (tree_choice.empty()) tree_choice = "chain-input";
  } else {
    tp::fail(tp::Errc::bad_argument, "--scheme must be jacobi or gauss-seidel");
  }
  const tp::TtmTree tree = tp::build_tree(s, strategy_from_name(tree_choice));

  // same sequence as the reference (random start, error, then sweep / error pairs); the tensor is uploaded once
  // and every sweep and error evaluation runs on the device
  const std::string init = a.get("--init", "random");
  if (init != "random" && init != "sthosvd") tp::fail(tp::Errc::bad_argument, "--init must be random or sthosvd");
  const tp::Decomposition start = init == "sthosvd" ? tp::sthosvd(t, s) : tp::random_decomposition(t, s, seed);
  tp::json steps = tp::json::array();
  std::string text;
  char line[160];
  std::snprintf(line, sizeof line, "start: error %.12f\n", tp::reconstruction_error(t, start));
  text += line;
  // --procs P: the paper's block distribution on P GPUs of this box (rank p on device p modulo the device count:
  // with fewer devices than ranks several ranks share one, which is only useful for trying the path out)
  const u64 procs = a.has("--procs") ? parse_u64(a.get("--procs"), "--procs") : 1;
  std::unique_ptr<tp::GridHooi> grid_engine;
  std::unique_ptr<tp::DeviceHooi> engine;
  tp::json grid_report;
  if (procs > 1 || a.has("--grid")) {
    if (kind != tp::SweepKind::jacobi) tp::fail(tp::Errc::bad_argument, "--procs runs the jacobi scheme only");
    tp::DynamicGridScheme scheme;
    if (a.flag("--dynamic")) {
      scheme = tp::optimal_dynamic_scheme(tree, s, procs).scheme;
    } else if (a.has("--grid")) {
      tp::Grid g;
      std::string item;
      for (const char c : a.get("--grid") + "x") {
        if (c == 'x') {
          g.q.push_back(parse_u64(item, "--grid"));
          item.clear();
        } else {
          item.push_back(c);
        }
      }
      tp::validate_grid(g, s, procs);
      scheme = tp::uniform_scheme(tree, g);
    } else {
      scheme = tp::uniform_scheme(tree, tp::optimal_static_grid(tree, s, procs).grid);
    }
    int device_count = 1;
    tp::detail::check(tp_device_count(&device_count));
    std::vector<int> devices;
    for (u64 p = 0; p < procs; ++p) devices.push_back(static_cast<int>(p % static_cast<u64>(device_count)));
    grid_engine = std::make_unique<tp::GridHooi>(t, s, tree, scheme, devices);
    grid_engine->set_factors(start.factors);
    grid_report = tp::json::object({{"procs", tp::json(procs)},
                                    {"devices", tp::json(static_cast<u64>(std::min<u64>(procs, device_count)))},
                                    {"scheme", tp::scheme_to_json(scheme)},
                                    {"model_volume", tp::json(tp::scheme_volume(tree, s, scheme, procs).total)}});
    std::snprintf(line, sizeof line, "grid: %llu ranks on %d device(s), model volume %llu elements per sweep\n",
                  static_cast<unsigned long long>(procs), std::min<int>(static_cast<int>(procs), device_count),
                  static_cast<unsigned long long>(tp::scheme_volume(tree, s, scheme, procs).total));
    text += line;
  } else {
    engine = std::make_unique<tp::DeviceHooi>(t, s, tree, kind);
    engine->set_factors(start.factors);
  }
  double final_error = tp::reconstruction_error(t, start);
  for (u64 i = 0; i < sweeps; ++i) {
    const tp::SweepStats stats = grid_engine ? grid_engine->sweep() : engine->sweep();
    // on the grid the error comes from the norms (orthonormal factors): no rank holds the whole tensor
    const double err = grid_engine ? grid_engine->fit_from_norms() : engine->reconstruction_error();
    final_error = err;
    steps.push_back(tp::json::object({{"sweep", tp::json(i + 1)},
                                      {"error", tp::json(err)},
                                      {"tree_macs", tp::json(stats.tree_macs)},
                                      {"core_macs", tp::json(stats.core_macs)},
                                      {"peak_live", tp::json(stats.peak_live)},
                                      {"degenerate", tp::json(stats.degenerate)}}));
    std::snprintf(line, sizeof line, "sweep %llu: error %.12f, tree macs %llu, peak live %d%s\n",
                  static_cast<unsigned long long>(i + 1), err, static_cast<unsigned long long>(stats.tree_macs),
                  stats.peak_live, stats.degenerate ? " (degenerate cut)" : "");
    text += line;
  }
  tp::json report = tp::json::object({{"spec", tp::spec_to_json(s)},
                                      {"tree", tp::json(tree_choice)},
                                      {"scheme", tp::json(scheme_name)},
                                      {"sweeps", steps},
                                      {"final_error", tp::json(final_error)}});
  if (grid_engine) report["grid"] = grid_report;
  emit(report.dump(2) + "\n", text, a);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    print_usage(nullptr);
    return 1;
  }
  const std::string first = argv[1];
  if (first == "--help" || first == "-h") {
    print_usage(nullptr);
    return 0;
  }
  const Command* cmd = nullptr;
  for (const Command& c : commands())
    if (first == c.name) cmd = &c;
  if (!cmd) {
    std::fprintf(stderr, "error: unknown subcommand %s%s\n", first.c_str(),
                 first == "bench" ? " (corpus statistics are not part of the B200 engine)" : "");
    return 1;
  }
  Args args;
  for (int i = 2; i < argc; ++i) {
    const std::string name = argv[i];
    if (name == "--help" || name == "-h") {
      print_usage(cmd);
      return 0;
    }
    const OptionSpec* opt = nullptr;
    for (const OptionSpec& o : cmd->options)
      if (name == o.name) opt = &o;
    if (!opt) {
      std::fprintf(stderr, "error: %s does not take %s\n", cmd->name, name.c_str());
      return 1;
    }
    if (opt->flag) {
      args.flags.insert(name);
    } else {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "error: %s needs a value\n", name.c_str());
        return 1;
      }
      args.values[name] = argv[++i];
    }
  }
  try {
    if (first == "plan") return cmd_plan(args);
    if (first == "simulate") return cmd_simulate(args);
    if (first == "gen-tensor") return cmd_gen_tensor(args);
    if (first == "hooi") return cmd_hooi(args);
  } catch (const tp::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 1;
}
