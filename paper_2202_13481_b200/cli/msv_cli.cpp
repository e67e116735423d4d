// msv — the experiment runner of SPEC.md's `cli` module: `run`, `plan`
// and `sweep` over one JSON config file. The reference ships only a stub
// (proj/tools/main.cpp:1), so this program is the specification's runner, written
// against nothing but the public header API that the reference (proj/include/migserve)
// and this repo's drop-in (include/migserve) share:
//
//   product   g++ ... -Iinclude msv_cli.cpp -lmsv      -> paper_2202_13481_b200/msv
//             every sample_trace / run / tail_latency / LBT call executes on the B200
//   checker   g++ ... -I/root/reference/proj/include    -> oracle/_ref/msv_cli_ref
//             (oracle/build_oracle.py; test infrastructure: the reference CPU engine)
//
// tests/ run both on the same configs and require byte-identical output trees.
//
// Usage:  msv run|plan|sweep <config.json> [--out DIR] [--set a.b=VALUE]...
// Output root: a relative output directory is resolved under $MSV_OUTPUT_ROOT if set.
// Exit codes: 0 ok, 1 validation (config or library input errors, with the
// offending field path), 2 runtime (I/O, device).
//
// Config format (every key optional unless noted; unknown keys are rejected):
//   profile  {"preset": "light"|"medium"|"heavy"|"mobilenet"|"resnet50"|"bert_base"}
//            | {"synthetic": {work_per_sample, fixed_overhead, parallelism_per_sample, util_cap}}
//            | {"csv": path, "model": name};  "sizes" [1,2,3,4,7], "b_max" 32 (synthetic)
//   workload {"mu" 1.0, "sigma" 1.0 | "pmf": [...], "rate_qps" (run), "duration_ms" 20000,
//             "seeds" [1,2,3], "trace_jsonl": path (run: replay instead of sampling)}
//   server   {"num_gpus" 1, "gpcs_per_gpu" 7, "total_gpcs" num_gpus*gpcs_per_gpu}
//   sla      {"multiplier" 1.5 | "target_ms", "alpha" 1, "beta" 1, "tail_p" 0.95}
//   paris    {"knee_threshold" 0.8}
//   engine   {"warmup_fraction" 0.1, "noise_sigma" 0, "noise_seed" 1, "check_wait_consistency" false}
//   search   {"duration_ms" = workload, "seeds" = workload, "rel_tol" 0.01, "lambda_min" 1,
//             "max_doublings" 24, "pinned_rate_qps", "curve_fractions" [...]}   (sweep, gpu(max))
//   designs  (required) [{"plan": "paris"|"gpu(K)"|"gpu(max)"|"random(SEED)"|{"gpus": [[...]]},
//                         "scheduler": "elsa"|"fifs", "segment_routing" false, "label"}]
//   output   {"dir" "msv_out", "per_query_csv" true}
#include <algorithm>
#include <cmath>
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

#include <migserve/engine.hpp>
#include <migserve/errors.hpp>
#include <migserve/metrics.hpp>
#include <migserve/paris.hpp>
#include <migserve/profile.hpp>
#include <migserve/workload.hpp>

// This repo's engine adds a batch entry point (include/migserve/grid.hpp: one device launch
// sequence for many independent simulations). When it is there, sweep's rate searches run
// in lockstep and its tail evaluations go to the device as one grid; results are the same
// numbers the per-simulation calls give (the GPU tests compare the output trees).
#if __has_include(<migserve/grid.hpp>)
#include <migserve/grid.hpp>
#define MSV_CLI_BATCHED 1
#endif

namespace fs = std::filesystem;
using nlohmann::json;
using namespace migserve;

namespace {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

[[noreturn]] void bad(const std::string& path, const std::string& what) {
    throw ConfigError("config: " + path + ": " + what);
}

// A config object being read: every value taken (or defaulted) is written to the
// resolved copy, and keys nobody read are rejected by done().
class Section {
public:
    Section(const json* src, json* dst, std::string path) : src_(src), dst_(dst), path_(std::move(path)) {
        if (src_ && !src_->is_object()) bad(path_.empty() ? "<root>" : path_, "must be an object");
        if (!dst_->is_object()) *dst_ = json::object();
    }

    std::string at(const std::string& key) const { return path_.empty() ? key : path_ + "." + key; }
    bool has(const std::string& key) const { return src_ && src_->contains(key); }
    const json& raw(const std::string& key) {
        used_.insert(key);
        return src_->at(key);
    }
    void echo(const std::string& key, const json& v) { (*dst_)[key] = v; }

    double number(const std::string& key, std::optional<double> def) {
        if (!has(key)) {
            if (!def) bad(at(key), "missing");
            (*dst_)[key] = *def;
            return *def;
        }
        const json& v = raw(key);
        if (!v.is_number()) bad(at(key), "must be a number");
        double x = v.get<double>();
        if (!std::isfinite(x)) bad(at(key), "must be finite");
        (*dst_)[key] = v;
        return x;
    }
    double positive(const std::string& key, std::optional<double> def) {
        double x = number(key, def);
        if (!(x > 0.0)) bad(at(key), "must be > 0");
        return x;
    }
    long long integer(const std::string& key, std::optional<long long> def, long long lo) {
        if (!has(key)) {
            if (!def) bad(at(key), "missing");
            (*dst_)[key] = *def;
            return *def;
        }
        const json& v = raw(key);
        if (!v.is_number_integer()) bad(at(key), "must be an integer");
        long long x = v.get<long long>();
        if (x < lo) bad(at(key), "must be >= " + std::to_string(lo));
        (*dst_)[key] = v;
        return x;
    }
    bool boolean(const std::string& key, bool def) {
        if (!has(key)) {
            (*dst_)[key] = def;
            return def;
        }
        const json& v = raw(key);
        if (!v.is_boolean()) bad(at(key), "must be true or false");
        (*dst_)[key] = v;
        return v.get<bool>();
    }
    std::string string(const std::string& key, std::optional<std::string> def) {
        if (!has(key)) {
            if (!def) bad(at(key), "missing");
            (*dst_)[key] = *def;
            return *def;
        }
        const json& v = raw(key);
        if (!v.is_string()) bad(at(key), "must be a string");
        (*dst_)[key] = v;
        return v.get<std::string>();
    }
    std::vector<double> numbers(const std::string& key, std::vector<double> def) {
        if (!has(key)) {
            (*dst_)[key] = def;
            return def;
        }
        const json& v = raw(key);
        if (!v.is_array()) bad(at(key), "must be an array of numbers");
        std::vector<double> out;
        for (size_t i = 0; i < v.size(); ++i) {
            if (!v[i].is_number() || !std::isfinite(v[i].get<double>()))
                bad(at(key) + "[" + std::to_string(i) + "]", "must be a finite number");
            out.push_back(v[i].get<double>());
        }
        (*dst_)[key] = v;
        return out;
    }
    std::vector<uint64_t> seeds(const std::string& key, std::vector<uint64_t> def) {
        if (!has(key)) {
            (*dst_)[key] = def;
            return def;
        }
        const json& v = raw(key);
        if (!v.is_array() || v.empty()) bad(at(key), "must be a non-empty array of seeds");
        std::vector<uint64_t> out;
        for (size_t i = 0; i < v.size(); ++i) {
            if (!v[i].is_number_unsigned() && !(v[i].is_number_integer() && v[i].get<long long>() >= 0))
                bad(at(key) + "[" + std::to_string(i) + "]", "must be a non-negative integer");
            out.push_back(v[i].get<uint64_t>());
        }
        (*dst_)[key] = v;
        return out;
    }
    Section sub(const std::string& key) {
        const json* s = nullptr;
        if (has(key)) s = &raw(key);
        return Section(s, &(*dst_)[key], at(key));
    }
    void done() const {
        if (!src_) return;
        for (auto it = src_->begin(); it != src_->end(); ++it)
            if (!used_.count(it.key())) bad(at(it.key()), "unknown field");
    }

private:
    const json* src_;
    json* dst_;
    std::string path_;
    std::set<std::string> used_;
};

struct Design {
    std::string label;
    std::string plan_spec;  // "paris", "gpu(K)", "gpu(max)", "random(S)", "explicit"
    int k = 0;              // gpu(K)
    uint64_t random_seed = 0;
    json explicit_plan;
    SchedulerKind scheduler = SchedulerKind::Elsa;
    bool segment_routing = false;
    std::string where;      // designs[i], for error messages
    PartitionPlan plan;
    std::optional<LbtResult> lbt;  // gpu(max): the winning search, reused by sweep
};

struct Experiment {
    json resolved;
    std::optional<ProfileTable> table;
    std::optional<BatchDistribution> dist;
    SlaConfig sla;
    double sla_multiplier = 1.5;
    double tail_p = 0.95;
    int num_gpus = 1, gpcs_per_gpu = 7, total_gpcs = 7;
    double knee_threshold = 0.8;
    std::optional<double> rate_qps;
    double duration_ms = 20000.0;
    std::vector<uint64_t> seeds{1, 2, 3};
    std::optional<QueryTrace> trace;
    EngineOptions engine;
    LbtOptions lbt;
    std::optional<double> pinned_rate_qps;
    std::vector<double> curve_fractions;
    std::vector<Design> designs;
    std::string out_dir;
    bool per_query_csv = true;
    std::optional<ParisResult> paris;
};

const std::map<std::string, SyntheticProfileParams>& presets() {
    // Model classes as named synthetic presets; the same values as
    // paper_2202_13481_b200/workloads.py.
    static const std::map<std::string, SyntheticProfileParams> p = {
        {"mobilenet", {0.4, 0.5, 0.15, 0.95}}, {"light", {0.4, 0.5, 0.15, 0.95}},
        {"resnet50", {0.8, 0.8, 0.25, 0.95}},  {"medium", {0.8, 0.8, 0.25, 0.95}},
        {"bert_base", {4.0, 2.0, 0.40, 0.95}}, {"heavy", {4.0, 2.0, 0.40, 0.95}}};
    return p;
}

std::string sanitize(const std::string& s) {
    std::string o;
    for (char c : s) o += (std::isalnum(static_cast<unsigned char>(c)) || c == '.' || c == '-') ? c : '_';
    return o;
}

void parse_profile(Section s, Experiment& e) {
    int modes = s.has("preset") + s.has("synthetic") + s.has("csv");
    if (modes != 1) bad(s.at("preset"), "give exactly one of preset, synthetic, csv");
    if (s.has("csv")) {
        std::string path = s.string("csv", std::nullopt);
        std::optional<std::string> model;
        if (s.has("model")) model = s.string("model", std::nullopt);
        e.table = load_profile_csv_file(path, model);
    } else {
        SyntheticProfileParams p;
        std::string name = "synthetic";
        if (s.has("preset")) {
            name = s.string("preset", std::nullopt);
            auto it = presets().find(name);
            if (it == presets().end()) bad(s.at("preset"), "unknown preset '" + name + "'");
            p = it->second;
        } else {
            Section q = s.sub("synthetic");
            p.work_per_sample = q.number("work_per_sample", p.work_per_sample);
            p.fixed_overhead = q.number("fixed_overhead", p.fixed_overhead);
            p.parallelism_per_sample = q.number("parallelism_per_sample", p.parallelism_per_sample);
            p.util_cap = q.number("util_cap", p.util_cap);
            q.done();
        }
        std::vector<int> sizes;
        for (double k : s.numbers("sizes", {1, 2, 3, 4, 7})) {
            if (k != std::floor(k) || k < 1) bad(s.at("sizes"), "sizes must be positive integers");
            sizes.push_back(static_cast<int>(k));
        }
        int b_max = static_cast<int>(s.integer("b_max", 32, 1));
        e.table = synth_profile(p, sizes, b_max, name);
    }
    s.done();
}

void parse_workload(Section s, Experiment& e) {
    if (s.has("pmf")) {
        e.dist = BatchDistribution(s.numbers("pmf", {}));
    } else {
        double mu = s.number("mu", 1.0);
        double sigma = s.positive("sigma", 1.0);
        e.dist = lognormal_batch_pdf(mu, sigma, static_cast<int>(s.integer("b_max", e.table->b_max(), 1)));
    }
    if (s.has("rate_qps")) e.rate_qps = s.positive("rate_qps", std::nullopt);
    e.duration_ms = s.positive("duration_ms", 20000.0);
    e.seeds = s.seeds("seeds", {1, 2, 3});
    if (s.has("trace_jsonl")) e.trace = read_trace_jsonl_file(s.string("trace_jsonl", std::nullopt));
    s.done();
}

Design parse_design(Section s, const std::string& where) {
    Design d;
    d.where = where;
    if (!s.has("plan")) bad(s.at("plan"), "missing");
    const json& p = s.raw("plan");
    s.echo("plan", p);
    if (p.is_object()) {
        d.plan_spec = "explicit";
        d.explicit_plan = p;
        if (!s.has("label")) bad(s.at("label"), "required for an explicit plan");
    } else if (p.is_string()) {
        std::string v = p.get<std::string>();
        auto arg = [&](const std::string& head) -> std::optional<std::string> {
            if (v.size() > head.size() + 2 && v.rfind(head + "(", 0) == 0 && v.back() == ')')
                return v.substr(head.size() + 1, v.size() - head.size() - 2);
            return std::nullopt;
        };
        auto digits = [&](const std::string& a) {
            if (a.empty() || a.size() > 18 || !std::all_of(a.begin(), a.end(), ::isdigit))
                bad(s.at("plan"), "bad plan spec '" + v + "'");
            return std::stoull(a);
        };
        if (v == "paris") {
            d.plan_spec = "paris";
        } else if (v == "gpu(max)") {
            d.plan_spec = "gpu(max)";
        } else if (auto a = arg("gpu")) {
            d.plan_spec = "gpu(K)";
            d.k = static_cast<int>(digits(*a));
        } else if (auto a2 = arg("random")) {
            d.plan_spec = "random(S)";
            d.random_seed = digits(*a2);
        } else {
            bad(s.at("plan"), "unknown plan '" + v + "' (paris, gpu(K), gpu(max), random(SEED) or {\"gpus\": ...})");
        }
    } else {
        bad(s.at("plan"), "must be a string or an object");
    }
    std::string sched = s.string("scheduler", std::string("elsa"));
    if (sched != "elsa" && sched != "fifs") bad(s.at("scheduler"), "unknown scheduler '" + sched + "' (elsa, fifs)");
    d.scheduler = scheduler_from_string(sched);
    d.segment_routing = s.boolean("segment_routing", false);
    std::string plan_label = p.is_string() ? p.get<std::string>() : std::string();
    d.label = s.string("label", plan_label + "+" + sched);
    s.done();
    return d;
}

Experiment parse(const json& cfg) {
    Experiment e;
    Section root(&cfg, &e.resolved, "");
    parse_profile(root.sub("profile"), e);
    parse_workload(root.sub("workload"), e);
    {
        Section s = root.sub("server");
        e.num_gpus = static_cast<int>(s.integer("num_gpus", 1, 1));
        e.gpcs_per_gpu = static_cast<int>(s.integer("gpcs_per_gpu", 7, 1));
        e.total_gpcs = static_cast<int>(s.integer("total_gpcs", e.num_gpus * e.gpcs_per_gpu, 1));
        s.done();
    }
    {
        Section s = root.sub("sla");
        e.tail_p = s.number("tail_p", 0.95);
        if (!(e.tail_p > 0.0 && e.tail_p < 1.0)) bad(s.at("tail_p"), "must be in (0, 1)");
        if (s.has("target_ms")) {
            e.sla.sla_target_ms = s.positive("target_ms", std::nullopt);
            e.sla_multiplier = 0.0;
        } else {
            e.sla_multiplier = s.positive("multiplier", 1.5);
            e.sla.sla_target_ms = derive_sla_target(*e.table, e.table->b_max(), e.sla_multiplier);
        }
        e.sla.alpha = s.number("alpha", 1.0);
        e.sla.beta = s.number("beta", 1.0);
        e.sla.validate();
        s.done();
    }
    {
        Section s = root.sub("paris");
        e.knee_threshold = s.number("knee_threshold", 0.8);
        s.done();
    }
    {
        Section s = root.sub("engine");
        e.engine.warmup_fraction = s.number("warmup_fraction", 0.1);
        e.engine.noise_sigma = s.number("noise_sigma", 0.0);
        e.engine.noise_seed = static_cast<uint64_t>(s.integer("noise_seed", 1, 0));
        e.engine.check_wait_consistency = s.boolean("check_wait_consistency", false);
        s.done();
    }
    {
        Section s = root.sub("search");
        e.lbt.duration_ms = s.positive("duration_ms", e.duration_ms);
        e.lbt.seeds = s.seeds("seeds", e.seeds);
        e.lbt.rel_tol = s.positive("rel_tol", 0.01);
        e.lbt.lambda_min = s.positive("lambda_min", 1.0);
        e.lbt.max_doublings = static_cast<int>(s.integer("max_doublings", 24, 0));
        e.lbt.tail_p = e.tail_p;
        e.lbt.warmup_fraction = e.engine.warmup_fraction;
        if (s.has("pinned_rate_qps")) e.pinned_rate_qps = s.positive("pinned_rate_qps", std::nullopt);
        e.curve_fractions = s.numbers("curve_fractions", {0.2, 0.4, 0.6, 0.8, 0.9, 1.0, 1.1, 1.2});
        for (double f : e.curve_fractions)
            if (!(f > 0.0)) bad(s.at("curve_fractions"), "fractions must be > 0");
        s.done();
    }
    {
        if (!root.has("designs")) bad("designs", "missing");
        const json& ds = root.raw("designs");
        if (!ds.is_array() || ds.empty()) bad("designs", "must be a non-empty array");
        json& out = e.resolved["designs"] = json::array();
        std::set<std::string> labels;
        for (size_t i = 0; i < ds.size(); ++i) {
            std::string where = "designs[" + std::to_string(i) + "]";
            out.push_back(json::object());
            Design d = parse_design(Section(&ds[i], &out.back(), where), where);
            if (!labels.insert(d.label).second) bad(where + ".label", "duplicate design label '" + d.label + "'");
            e.designs.push_back(std::move(d));
        }
    }
    {
        Section s = root.sub("output");
        e.out_dir = s.string("dir", std::string("msv_out"));
        e.per_query_csv = s.boolean("per_query_csv", true);
        s.done();
    }
    if (root.has("derived")) root.raw("derived");  // an echoed resolved config re-runs as is
    e.resolved.erase("derived");
    root.done();
    return e;
}

const ParisResult& paris(Experiment& e) {
    if (!e.paris) e.paris = paris_plan(*e.table, *e.dist, e.total_gpcs, e.num_gpus, e.gpcs_per_gpu, e.knee_threshold);
    return *e.paris;
}

// Resolve every design's plan; gpu(max) runs best_homogeneous (metrics.hpp:183-209),
// which simulates, so `plan` skips it.
void resolve_plans(Experiment& e, bool simulate) {
    for (Design& d : e.designs) {
        if (d.plan_spec == "paris") {
            d.plan = paris(e).plan;
        } else if (d.plan_spec == "gpu(K)") {
            d.plan = homogeneous_plan(d.k, e.total_gpcs, e.num_gpus, e.gpcs_per_gpu);
        } else if (d.plan_spec == "random(S)") {
            d.plan = random_plan(e.num_gpus, e.gpcs_per_gpu, d.random_seed, e.table->sizes());
        } else if (d.plan_spec == "explicit") {
            d.plan = PartitionPlan::from_json(d.explicit_plan);
        } else if (d.plan_spec == "gpu(max)" && simulate) {
            BestHomogeneous b = best_homogeneous(*e.table, *e.dist, e.sla, e.total_gpcs, e.num_gpus, e.gpcs_per_gpu,
                                                 e.lbt);
            d.plan = b.plan;
            d.k = b.k;
            d.lbt = b.lbt;
        }
    }
}

EngineOptions options_for(Experiment& e, const Design& d) {
    EngineOptions o = e.engine;
    if (d.segment_routing) {  // route by the PARIS planning segments (engine.hpp:41-42, :197-206)
        o.segment_routing = true;
        o.routing_segments = paris(e).segments;
    }
    return o;
}

json paris_json(const ParisResult& r) {
    json knees = json::object();
    for (auto [k, b] : r.knees) knees[std::to_string(k)] = b;
    json segs = json::array();
    for (const BatchSegment& s : r.segments) segs.push_back({{"k", s.k.gpcs}, {"first", s.first}, {"last", s.last}});
    json ratios = json::array();
    for (const RatioEntry& x : r.ratios.entries)
        ratios.push_back({{"k", x.k.gpcs}, {"ratio", x.ratio}, {"segment_mass", x.segment_mass}});
    json counts = json::array();
    for (const auto& [k, n] : r.counts.counts) counts.push_back({{"k", k.gpcs}, {"real_count", n}});
    return json{{"knees", knees},
                {"segments", segs},
                {"ratios", ratios},
                {"counts", counts},
                {"weighted_sum", r.counts.weighted_sum},
                {"normalizer", r.counts.normalizer},
                {"plan", r.plan.to_json()}};
}

json derived(Experiment& e) {
    json d{{"sla_target_ms", e.sla.sla_target_ms}, {"profile_model", e.table->model_name()}};
    json ds = json::array();
    for (const Design& x : e.designs) {
        json j{{"label", x.label}, {"scheduler", to_string(x.scheduler)}};
        if (x.plan_spec == "gpu(max)" && x.k == 0) {
            j["plan"] = nullptr;  // chosen by simulation (run / sweep)
        } else {
            j["plan"] = x.plan.to_json();
            if (x.plan_spec == "gpu(max)") j["gpu_max_k"] = x.k;
        }
        ds.push_back(j);
    }
    d["designs"] = ds;
    bool any_paris = std::any_of(e.designs.begin(), e.designs.end(),
                                 [](const Design& x) { return x.plan_spec == "paris" || x.segment_routing; });
    if (any_paris) d["paris"] = paris_json(paris(e));
    return d;
}

void write_file(const fs::path& p, const std::string& text) {
    std::ofstream f(p, std::ios::binary);
    if (!f) throw std::runtime_error("cannot write " + p.string());
    f << text;
    if (!f) throw std::runtime_error("write failed: " + p.string());
}

fs::path output_dir(const Experiment& e) {
    fs::path p(e.out_dir);
    const char* root = std::getenv("MSV_OUTPUT_ROOT");
    if (p.is_relative() && root && *root) p = fs::path(root) / p;
    fs::create_directories(p);
    return p;
}

// Mean of per-seed tails in seed order over the seeds with measured samples
// (the reference's detail::mean_tail_at_rate, metrics.hpp:57-75), for every
// (design, rate) probe.
std::vector<double> mean_tails(const Experiment& e, const std::vector<std::pair<const Design*, double>>& probes) {
    std::vector<double> out(probes.size(), 0.0);
#ifdef MSV_CLI_BATCHED
    std::vector<GridCell> cells;
    for (const auto& [d, rate] : probes)
        for (uint64_t seed : e.lbt.seeds) {
            GridCell c;
            c.plan = &d->plan;
            c.scheduler = d->scheduler;
            c.table = &*e.table;
            c.dist = &*e.dist;
            c.sla = e.sla;
            c.rate_qps = rate;
            c.duration_ms = e.lbt.duration_ms;
            c.seed = seed;
            c.warmup_fraction = e.lbt.warmup_fraction;
            cells.push_back(c);
        }
    std::vector<GridCellResult> res = run_grid(cells, {e.tail_p});
    for (size_t i = 0, c = 0; i < probes.size(); ++i) {
        double sum = 0.0;
        int used = 0;
        for (size_t j = 0; j < e.lbt.seeds.size(); ++j, ++c) {
            if (res[c].measured_queries == 0) continue;
            sum += res[c].tails[0];
            ++used;
        }
        out[i] = used == 0 ? 0.0 : sum / static_cast<double>(used);
    }
#else
    for (size_t i = 0; i < probes.size(); ++i) {
        const auto& [d, rate] = probes[i];
        double sum = 0.0;
        int used = 0;
        for (uint64_t seed : e.lbt.seeds) {
            QueryTrace trace = sample_trace(*e.dist, rate, e.lbt.duration_ms, seed);
            EngineOptions eng;
            eng.warmup_fraction = e.lbt.warmup_fraction;
            SimReport rep = run(d->plan, d->scheduler, trace, *e.table, e.sla, eng);
            std::vector<double> samples = rep.latency_samples();
            if (samples.empty()) continue;
            sum += tail_latency(std::move(samples), e.tail_p);
            ++used;
        }
        out[i] = used == 0 ? 0.0 : sum / static_cast<double>(used);
    }
#endif
    return out;
}

// latency_bounded_throughput (metrics.hpp:81-120) for every design still without one.
void search_all(Experiment& e) {
#ifdef MSV_CLI_BATCHED
    std::vector<detail::LbtSearch> searches;
    std::vector<Design*> owners;
    for (Design& d : e.designs) {
        if (d.lbt) continue;
        detail::LbtSearch s;
        s.plan = &d.plan;
        s.scheduler = d.scheduler;
        s.table = &*e.table;
        s.cfg = e.sla;
        s.dist = &*e.dist;
        s.opt = e.lbt;
        searches.push_back(s);
        owners.push_back(&d);
    }
    if (!searches.empty()) detail::run_lockstep(searches);
    for (size_t i = 0; i < owners.size(); ++i) owners[i]->lbt = searches[i].result;
#else
    for (Design& d : e.designs)
        if (!d.lbt) d.lbt = latency_bounded_throughput(d.plan, d.scheduler, *e.table, e.sla, *e.dist, e.lbt);
#endif
}

int cmd_plan(Experiment& e) {
    resolve_plans(e, false);
    json out = derived(e);
    out["paris"] = paris_json(paris(e));
    std::cout << out.dump(2) << "\n";
    return 0;
}

// run: every design x seed simulated at workload.rate_qps (or on the replayed trace);
// per-run report JSON (+ per-query CSV), a summary CSV, the resolved config.
int cmd_run(Experiment& e) {
    if (!e.rate_qps && !e.trace) bad("workload.rate_qps", "missing (run needs a rate or a trace_jsonl)");
    resolve_plans(e, true);
    fs::path out = output_dir(e);
    fs::create_directories(out / "reports");
    std::ostringstream sum;
    sum << "label,scheduler,instances,used_gpcs,rate_qps,seeds,queries,violations,measured_queries,"
           "measured_violations,tail_p,mean_tail_ms,mean_p99_ms\n";
    std::vector<uint64_t> seeds = e.trace ? std::vector<uint64_t>{e.trace->seed} : e.seeds;
    for (const Design& d : e.designs) {
        EngineOptions opt = options_for(e, d);
        long long total = 0, viol = 0, meas = 0, mviol = 0;
        double tail_sum = 0.0, p99_sum = 0.0;
        int used = 0;
        for (uint64_t seed : seeds) {
            QueryTrace trace = e.trace ? *e.trace : sample_trace(*e.dist, *e.rate_qps, e.duration_ms, seed);
            SimReport r = run(d.plan, d.scheduler, trace, *e.table, e.sla, opt);
            std::string stem = sanitize(d.label) + "__seed" + std::to_string(seed);
            write_file(out / "reports" / (stem + ".json"), report_to_json(r).dump(2) + "\n");
            if (e.per_query_csv) {
                std::ostringstream csv;
                write_query_csv(r, csv);
                write_file(out / "reports" / (stem + ".csv"), csv.str());
            }
            total += r.total_queries;
            viol += r.violations;
            meas += r.measured_queries;
            mviol += r.measured_violations;
            std::vector<double> s = r.latency_samples();
            if (s.empty()) continue;
            tail_sum += tail_latency(s, e.tail_p);
            p99_sum += tail_latency(std::move(s), 0.99);
            ++used;
        }
        sum << d.label << ',' << to_string(d.scheduler) << ',' << d.plan.total_instances() << ','
            << d.plan.used_gpcs() << ',' << format_double(e.trace ? 0.0 : *e.rate_qps) << ',' << seeds.size() << ','
            << total << ',' << viol << ',' << meas << ',' << mviol << ',' << format_double(e.tail_p) << ','
            << format_double(used ? tail_sum / used : 0.0) << ',' << format_double(used ? p99_sum / used : 0.0)
            << '\n';
    }
    write_file(out / "summary.csv", sum.str());
    json resolved = e.resolved;
    resolved["derived"] = derived(e);
    write_file(out / "resolved_config.json", resolved.dump(2) + "\n");
    std::cout << (out / "summary.csv").string() << "\n";
    return 0;
}

// sweep: latency-bounded throughput per design (metrics.hpp:81-120), the tail at a
// common pinned rate, compare() against gpu(7)+fifs (metrics.hpp:146-170) -> summary CSV,
// and the tail-latency vs offered-load curve per design (Fig. 9 axes) -> plot-data CSV.
int cmd_sweep(Experiment& e) {
    bool has_base = false;
    for (const Design& d : e.designs) {
        has_base |= d.label == kBaselineLabel;
        if (d.segment_routing) bad(d.where + ".segment_routing", "not supported by sweep (the rate search has no engine options)");
    }
    if (!has_base) bad("designs", std::string("sweep normalises to ") + kBaselineLabel + ", which is not listed");
    if (e.engine.noise_sigma != 0.0 || e.engine.check_wait_consistency)
        bad("engine", "sweep runs the rate search with default engine options (noise_sigma 0, no wait check)");
    resolve_plans(e, true);
    search_all(e);
    std::vector<DesignPoint> points;
    for (Design& d : e.designs) {
        DesignPoint p;
        p.label = d.label;
        p.scheduler = d.scheduler;
        p.plan = d.plan;
        p.seeds = e.lbt.seeds;
        p.lbt = *d.lbt;
        points.push_back(std::move(p));
    }
    double pinned = 0.0, top = 0.0;
    if (e.pinned_rate_qps) {
        pinned = *e.pinned_rate_qps;
    } else {  // the largest load every design sustains within the SLA
        for (const DesignPoint& p : points)
            if (p.lbt.qps > 0.0) pinned = pinned == 0.0 ? p.lbt.qps : std::min(pinned, p.lbt.qps);
    }
    for (const DesignPoint& p : points) top = std::max(top, p.lbt.qps);
    // every tail the outputs need, evaluated together: the pinned-rate tails, then the curves
    std::vector<std::pair<const Design*, double>> probes;
    for (const Design& d : e.designs)
        if (pinned > 0.0) probes.emplace_back(&d, pinned);
    size_t curve0 = probes.size();
    for (const Design& d : e.designs)
        for (double f : e.curve_fractions)
            if (f * top > 0.0) probes.emplace_back(&d, f * top);
    std::vector<double> tails = mean_tails(e, probes);
    for (size_t i = 0; i < points.size(); ++i) {
        points[i].rate_qps = pinned;
        points[i].tail_ms_at_rate = pinned > 0.0 ? tails[i] : 0.0;
    }
    std::vector<ComparisonRow> rows = compare(points);
    fs::path out = output_dir(e);
    std::ostringstream sum;
    sum << "label,scheduler,instances,used_gpcs,lbt_qps,infeasible_at_min,sims_run,pinned_rate_qps,tail_p,tail_ms,"
           "norm_lbt,norm_tail\n";
    for (size_t i = 0; i < rows.size(); ++i) {
        const DesignPoint& p = points[i];
        sum << rows[i].label << ',' << to_string(p.scheduler) << ',' << p.plan.total_instances() << ','
            << p.plan.used_gpcs() << ',' << format_double(rows[i].lbt_qps) << ','
            << (p.lbt.infeasible_at_min ? 1 : 0) << ',' << p.lbt.sims_run << ',' << format_double(p.rate_qps) << ','
            << format_double(e.tail_p) << ',' << format_double(rows[i].tail_ms) << ','
            << format_double(rows[i].norm_lbt) << ',' << format_double(rows[i].norm_tail) << '\n';
    }
    write_file(out / "summary.csv", sum.str());
    std::ostringstream plot;
    plot << "label,offered_fraction,offered_qps,tail_p,mean_tail_ms,sla_target_ms\n";
    size_t next = curve0;
    for (const Design& d : e.designs)
        for (double f : e.curve_fractions) {
            double rate = f * top;
            double t = rate > 0.0 ? tails[next++] : 0.0;
            plot << d.label << ',' << format_double(f) << ',' << format_double(rate) << ',' << format_double(e.tail_p)
                 << ',' << format_double(t) << ',' << format_double(e.sla.sla_target_ms) << '\n';
        }
    write_file(out / "plot_data.csv", plot.str());
    json resolved = e.resolved;
    resolved["derived"] = derived(e);
    write_file(out / "resolved_config.json", resolved.dump(2) + "\n");
    std::cout << (out / "summary.csv").string() << "\n";
    return 0;
}

int usage() {
    std::cerr << "usage: msv run|plan|sweep <config.json> [--out DIR] [--set key.path=VALUE]...\n";
    return 1;
}

// --set a.b.c=VALUE: VALUE parsed as JSON when it parses, else taken as a string.
void apply_set(json& cfg, const std::string& arg) {
    size_t eq = arg.find('=');
    if (eq == std::string::npos || eq == 0) throw ConfigError("--set: expected key.path=VALUE, got '" + arg + "'");
    std::string key = arg.substr(0, eq), val = arg.substr(eq + 1);
    json v = json::parse(val, nullptr, false);
    if (v.is_discarded()) v = val;
    json* node = &cfg;
    size_t pos = 0;
    for (;;) {
        size_t dot = key.find('.', pos);
        std::string part = key.substr(pos, dot == std::string::npos ? std::string::npos : dot - pos);
        if (part.empty()) throw ConfigError("--set: bad key '" + key + "'");
        if (!node->is_object()) throw ConfigError("--set: " + key + ": parent is not an object");
        if (dot == std::string::npos) {
            (*node)[part] = v;
            return;
        }
        node = &(*node)[part];
        if (node->is_null()) *node = json::object();
        pos = dot + 1;
    }
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 3) return usage();
        std::string verb = argv[1];
        if (verb != "run" && verb != "plan" && verb != "sweep") return usage();
        std::ifstream f(argv[2]);
        if (!f) throw ConfigError("config: cannot open " + std::string(argv[2]));
        json cfg = json::parse(f, nullptr, false);
        if (cfg.is_discarded()) throw ConfigError("config: " + std::string(argv[2]) + ": not valid JSON");
        for (int i = 3; i < argc; ++i) {
            std::string a = argv[i];
            if (a == "--out" && i + 1 < argc) {
                apply_set(cfg, "output.dir=" + json(std::string(argv[++i])).dump());
            } else if (a == "--set" && i + 1 < argc) {
                apply_set(cfg, argv[++i]);
            } else {
                return usage();
            }
        }
        Experiment e = parse(cfg);
        if (verb == "plan") return cmd_plan(e);
        if (verb == "run") return cmd_run(e);
        return cmd_sweep(e);
    } catch (const ConfigError& ex) {
        std::cerr << "msv: " << ex.what() << "\n";
        return 1;
    } catch (const ParamError& ex) {
        std::cerr << "msv: ParamError: " << ex.what() << "\n";
        return 1;
    } catch (const FormatError& ex) {
        std::cerr << "msv: FormatError: " << ex.what() << "\n";
        return 1;
    } catch (const ValidationError& ex) {
        std::cerr << "msv: ValidationError: " << ex.what() << "\n";
        return 1;
    } catch (const LookupError& ex) {
        std::cerr << "msv: LookupError: " << ex.what() << "\n";
        return 1;
    } catch (const InfeasibleError& ex) {
        std::cerr << "msv: InfeasibleError: " << ex.what() << "\n";
        return 1;
    } catch (const std::exception& ex) {
        std::cerr << "msv: runtime error: " << ex.what() << "\n";
        return 2;
    }
}
