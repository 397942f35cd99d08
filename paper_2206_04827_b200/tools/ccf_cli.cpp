// `cylspec` command-line driver over the B200 library (drop-in for the reference CLI,
// proj/tools/cylspec_main.cpp:67-386, and its run configuration, proj/src/runconfig.cpp):
//
//   cylspec heat|poisson|ns|transform [--config cfg.json] [--m M] [--n N] [--p P] [--steps S] [--h H]
//           [--alpha A] [--re RE] [--bdf B] [--tol T] [--out DIR] [--in FILE] [--seed S] [--case C]
//           [--output-every K]
//
// Same subcommands, flags, JSON config keys (flat object; CLI flags override file values), output
// files (CCF1 FieldFiles + manifest.json) and exit codes (0 ok, 2 config / domain error, 3 numerical
// or i/o failure with out/failure_manifest.json; CLI parse errors use the CLI11 codes 104 / 106 /
// 109). Restrictions of the B200 path surface as DomainError (exit 2): even m and n. `bench` (the
// paper's Table-1 comparison against collocation / finite-difference / dense baselines) is not part
// of this hot path; tools/heat_table1.py runs the spectral column.
#include <array>
#include <cctype>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>

#include "cylspec_b200.hpp"

namespace fs = std::filesystem;
using namespace cylspec;

namespace {

constexpr int kExitOk = 0, kExitConfig = 2, kExitNumerical = 3;
constexpr int kCliConversion = 104, kCliRequired = 106, kCliExtras = 109;  // CLI11 exit codes

// ---------------------------------------------------------------- minimal JSON (flat config objects)
struct JVal {
    enum Kind { NUL, NUM, STR, BOOL, ARR } kind = NUL;
    double num = 0;
    std::string str;
    bool b = false;
    std::vector<JVal> arr;
};

struct JParser {
    const std::string& s;
    size_t i = 0;
    [[noreturn]] void fail(const std::string& what) {
        throw ConfigError("config parse error: " + what + " at offset " + std::to_string(i));
    }
    void ws() {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    }
    bool eat(char c) {
        ws();
        if (i < s.size() && s[i] == c) {
            ++i;
            return true;
        }
        return false;
    }
    std::string string() {
        if (!eat('"')) fail("expected string");
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\' && i + 1 < s.size()) {
                const char e = s[++i];
                out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
            } else {
                out += s[i];
            }
            ++i;
        }
        if (i >= s.size()) fail("unterminated string");
        ++i;
        return out;
    }
    JVal value() {
        ws();
        JVal v;
        if (i >= s.size()) fail("unexpected end");
        if (s[i] == '"') {
            v.kind = JVal::STR;
            v.str = string();
        } else if (s[i] == '[') {
            ++i;
            v.kind = JVal::ARR;
            if (!eat(']')) {
                do v.arr.push_back(value());
                while (eat(','));
                if (!eat(']')) fail("expected ]");
            }
        } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 5, "false") == 0) {
            v.kind = JVal::BOOL;
            v.b = s[i] == 't';
            i += v.b ? 4 : 5;
        } else if (s.compare(i, 4, "null") == 0) {
            i += 4;
        } else {
            size_t end = 0;
            try {
                v.num = std::stod(s.substr(i), &end);
            } catch (...) {
                fail("bad value");
            }
            v.kind = JVal::NUM;
            i += end;
        }
        return v;
    }
    std::map<std::string, JVal> object() {
        std::map<std::string, JVal> o;
        if (!eat('{')) fail("expected object");
        if (eat('}')) return o;
        do {
            ws();
            const std::string k = string();
            if (!eat(':')) fail("expected :");
            o[k] = value();
        } while (eat(','));
        if (!eat('}')) fail("expected }");
        ws();
        if (i != s.size()) fail("trailing characters");
        return o;
    }
};

// ---------------------------------------------------------------- RunConfig (runconfig.hpp:14-39)
struct RunConfig {
    std::string problem;
    int m = 15, n = 15, p = 16;
    double alpha = 1.0, reynolds = 100.0, h = 0.01;
    int steps = 200, bdf_order = 4;
    double adi_tol = 1e-12;
    int output_every = 0;
    std::string bc_kind = "dirichlet_homogeneous", output_path = "out", input_path, case_name = "manufactured";
    unsigned long long seed = 0;
    bool exact_forcing = true, collocation_cache_lu = false;
    std::vector<int> bench_sizes = {7, 11, 15, 19}, bench_fd_sizes = {61};
    std::vector<std::string> bench_methods = {"spectral", "collocation", "fd", "dense"};
    int threads = 1;

    void validate() const {  // runconfig.cpp:8-21
        if (problem != "heat" && problem != "poisson" && problem != "ns" && problem != "bench" && problem != "transform")
            throw ConfigError("unknown problem: " + problem);
        if (m <= 0 || n <= 0 || p <= 0) throw ConfigError("grid sizes must be positive");
        if (!(h > 0)) throw ConfigError("h must be positive");
        if (!(adi_tol > 0) || adi_tol > 1e-2) throw ConfigError("adi_tol must lie in (0, 1e-2]");
        if (steps < 0) throw ConfigError("steps must be nonnegative");
        if (bdf_order < 1 || bdf_order > 4) throw ConfigError("bdf_order must be 1..4");
        if (bc_kind != "dirichlet_homogeneous" && bc_kind != "dirichlet_lifted")
            throw ConfigError("unknown bc kind: " + bc_kind);
        if (threads < 1) throw ConfigError("threads must be >= 1");
    }
};

RunConfig load_config(const std::string& path) {  // runconfig.cpp:23-60
    RunConfig cfg;
    if (path.empty()) return cfg;
    std::ifstream is(path);
    if (!is) throw ConfigError("cannot open config file: " + path);
    std::stringstream ss;
    ss << is.rdbuf();
    const std::string text = ss.str();
    JParser jp{text};
    const auto o = jp.object();
    auto type_err = [](const std::string& k) { throw ConfigError("config parse error: wrong type for " + k); };
    auto num = [&](const char* k, auto& out) {
        auto it = o.find(k);
        if (it == o.end()) return;
        if (it->second.kind != JVal::NUM) type_err(k);
        out = static_cast<std::decay_t<decltype(out)>>(it->second.num);
    };
    auto str = [&](const char* k, std::string& out) {
        auto it = o.find(k);
        if (it == o.end()) return;
        if (it->second.kind != JVal::STR) type_err(k);
        out = it->second.str;
    };
    auto boo = [&](const char* k, bool& out) {
        auto it = o.find(k);
        if (it == o.end()) return;
        if (it->second.kind != JVal::BOOL) type_err(k);
        out = it->second.b;
    };
    str("problem", cfg.problem);
    num("m", cfg.m);
    num("n", cfg.n);
    num("p", cfg.p);
    num("alpha", cfg.alpha);
    num("reynolds", cfg.reynolds);
    num("h", cfg.h);
    num("steps", cfg.steps);
    num("bdf_order", cfg.bdf_order);
    num("adi_tol", cfg.adi_tol);
    num("output_every", cfg.output_every);
    str("bc_kind", cfg.bc_kind);
    str("output_path", cfg.output_path);
    str("input_path", cfg.input_path);
    str("case", cfg.case_name);
    num("seed", cfg.seed);
    boo("exact_forcing", cfg.exact_forcing);
    boo("collocation_cache_lu", cfg.collocation_cache_lu);
    num("threads", cfg.threads);
    for (const char* k : {"bench_sizes", "bench_fd_sizes"}) {
        auto it = o.find(k);
        if (it == o.end()) continue;
        if (it->second.kind != JVal::ARR) type_err(k);
        auto& dst = std::string(k) == "bench_sizes" ? cfg.bench_sizes : cfg.bench_fd_sizes;
        dst.clear();
        for (const JVal& v : it->second.arr) dst.push_back(int(v.num));
    }
    return cfg;
}

// ---------------------------------------------------------------- manifest writer
std::string jnum(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}
std::string jstr(const std::string& v) {
    std::string o = "\"";
    for (char c : v) o += (c == '"' || c == '\\') ? std::string("\\") + c : std::string(1, c);
    return o + "\"";
}

struct Manifest {
    std::vector<std::pair<std::string, std::string>> kv;  // key -> serialized value (insertion order)
    void put(const std::string& k, const std::string& raw) { kv.emplace_back(k, raw); }
    std::string dump() const {
        std::string o = "{\n";
        for (size_t i = 0; i < kv.size(); ++i) o += "  " + jstr(kv[i].first) + ": " + kv[i].second + (i + 1 < kv.size() ? ",\n" : "\n");
        return o + "}\n";
    }
    void write(const fs::path& dir) const {
        std::ofstream os(dir / "manifest.json");
        os << dump();
    }
};

std::string config_json(const RunConfig& c) {
    std::string o = "{";
    auto add = [&](const std::string& k, const std::string& v) { o += (o.size() > 1 ? ", " : "") + jstr(k) + ": " + v; };
    add("problem", jstr(c.problem));
    add("m", std::to_string(c.m));
    add("n", std::to_string(c.n));
    add("p", std::to_string(c.p));
    add("alpha", jnum(c.alpha));
    add("reynolds", jnum(c.reynolds));
    add("h", jnum(c.h));
    add("steps", std::to_string(c.steps));
    add("bdf_order", std::to_string(c.bdf_order));
    add("adi_tol", jnum(c.adi_tol));
    add("output_every", std::to_string(c.output_every));
    add("bc_kind", jstr(c.bc_kind));
    add("output_path", jstr(c.output_path));
    add("input_path", jstr(c.input_path));
    add("case", jstr(c.case_name));
    add("seed", std::to_string(c.seed));
    add("exact_forcing", c.exact_forcing ? "true" : "false");
    add("threads", std::to_string(c.threads));
    return o + "}";
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ManufacturedHeat (bench.cpp:20-35)
double mh_exact(double r, double z, double th, double t) {
    return std::exp(-t) * std::cos(M_PI * z / 2) * (1 - r * r) * (1 + 0.5 * r * std::cos(th));
}
double mh_forcing(double r, double z, double th, double t, double alpha) {
    const double zz = std::cos(M_PI * z / 2);
    const double s = (1 - r * r) * (1 + 0.5 * r * std::cos(th));
    const double lap = std::exp(-t) * (-4.0 * zz * (1 + r * std::cos(th)) - M_PI * M_PI / 4.0 * zz * s);
    return -mh_exact(r, z, th, t) - alpha * lap;
}

GridField random_smooth_field(const GridSpec& spec, unsigned long long seed) {  // cylspec_main.cpp:54-65
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::array<double, 8> c;
    for (double& v : c) v = dist(rng);
    return sample(spec, [&](double r, double z, double th) {
        const double x = r * std::cos(th), y = r * std::sin(th);
        const double bump = (1 - r * r) * (1 - z * z);
        return bump * (c[0] + c[1] * x + c[2] * y + c[3] * z + c[4] * x * y + c[5] * x * z + c[6] * y * z +
                       c[7] * (x * x - y * y));
    });
}

int run_heat(const RunConfig& cfg) {
    const GridSpec spec(cfg.m, cfg.n, cfg.p);
    const fs::path outdir(cfg.output_path);
    fs::create_directories(outdir);
    GridField initial(spec);
    ForcingCallback forcing;
    const double alpha = cfg.alpha;
    if (cfg.case_name == "manufactured") {
        initial = sample(spec, [](double r, double z, double th) { return mh_exact(r, z, th, 0.0); });
        forcing = [spec, alpha](double t) {
            return sample(spec, [&](double r, double z, double th) { return mh_forcing(r, z, th, t, alpha); });
        };
    } else if (cfg.case_name == "decay") {
        initial = random_smooth_field(spec, cfg.seed);
    } else {
        throw ConfigError("unknown heat case: " + cfg.case_name);
    }
    HeatConfig hc;
    hc.spec = spec;
    hc.alpha = cfg.alpha;
    hc.h = cfg.h;
    hc.order = cfg.bdf_order;
    hc.adi_tol = cfg.adi_tol;
    hc.forcing_mode = cfg.exact_forcing ? ForcingMode::exact : ForcingMode::lagged;
    hc.output_every = cfg.output_every;
    const auto t0 = std::chrono::steady_clock::now();
    HeatRunResult run = heat_run(hc, initial, forcing, cfg.steps);
    const double sec = seconds_since(t0);
    Manifest mf;
    mf.put("command", jstr("heat"));
    mf.put("config", config_json(cfg));
    mf.put("timings", "{\"total_seconds\": " + jnum(sec) + ", \"per_step_seconds\": " +
                          jnum(cfg.steps ? sec / cfg.steps : 0) + "}");
    mf.put("worst_modal_residual", jnum(run.worst_residual));  // see HeatRunResult::worst_residual
    mf.put("modal_solver", jstr("fast diagonalization on the FP64 tensor cores"));
    mf.put("final_time", jnum(run.final_time));
    std::string outs = "[";
    for (size_t i = 0; i < run.snapshots.size(); ++i) {
        const std::string name = "snapshot_" + std::to_string(i) + ".ccf";
        write_field((outdir / name).string(), run.snapshots[i]);
        outs += std::string(i ? ", " : "") + "{\"path\": " + jstr(name) + ", \"time\": " + jnum(run.snapshot_times[i]) + "}";
    }
    if (cfg.case_name == "manufactured" && cfg.steps > 0) {
        const GridField ref =
            sample(spec, [&](double r, double z, double th) { return mh_exact(r, z, th, run.final_time); });
        double err = 0, scale = 0;
        for (size_t i = 0; i < ref.values.size(); ++i) {
            err = std::max(err, std::abs(run.snapshots.back().values[i] - ref.values[i]));
            scale = std::max(scale, std::abs(ref.values[i]));
        }
        mf.put("max_rel_error", jnum(scale > 0 ? err / scale : err));
    }
    mf.put("outputs", outs + "]");
    mf.write(outdir);
    return kExitOk;
}

int run_poisson(const RunConfig& cfg) {
    const GridSpec spec(cfg.m, cfg.n, cfg.p);
    const fs::path outdir(cfg.output_path);
    fs::create_directories(outdir);
    CoeffTensor f(spec);
    if (!cfg.input_path.empty()) {
        FieldVariant v = read_field(cfg.input_path);
        if (std::holds_alternative<GridField>(v)) f = analyze(std::get<GridField>(v));
        else f = std::get<CoeffTensor>(v);
        if (!(f.spec == spec)) throw ConfigError("input field dimensions disagree with the config");
    } else {  // f = lap T at t = 0 of the manufactured profile (cylspec_main.cpp:136-142)
        f = analyze(sample(spec, [](double r, double z, double th) {
            return -mh_exact(r, z, th, 0.0) - mh_forcing(r, z, th, 0.0, 1.0);
        }));
    }
    const auto t0 = std::chrono::steady_clock::now();
    CoeffTensor u = solve_poisson_3d(f, BoundaryCondition{}, cfg.adi_tol);
    const double sec = seconds_since(t0);
    write_field((outdir / "solution.ccf").string(), u);
    const GridField ug = synthesize(u);
    write_field((outdir / "solution_values.ccf").string(), ug);
    Manifest mf;
    mf.put("command", jstr("poisson"));
    mf.put("config", config_json(cfg));
    mf.put("timings", "{\"total_seconds\": " + jnum(sec) + "}");
    mf.put("outputs", "[\"solution.ccf\", \"solution_values.ccf\"]");
    if (cfg.input_path.empty()) {
        const GridField ref = sample(spec, [](double r, double z, double th) { return mh_exact(r, z, th, 0.0); });
        double err = 0;
        for (size_t i = 0; i < ug.values.size(); ++i) err = std::max(err, std::abs(ug.values[i] - ref.values[i]));
        mf.put("max_abs_error", jnum(err));
    }
    mf.write(outdir);
    return kExitOk;
}

int run_ns(const RunConfig& cfg) {
    const GridSpec spec(cfg.m, cfg.n, cfg.p);
    const fs::path outdir(cfg.output_path);
    fs::create_directories(outdir);
    // seeded smooth gauge-fixed initial scalars (cylspec_main.cpp:181-191), omega = curl_pt(v-scalars)
    std::mt19937_64 rng(cfg.seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    const double a0 = dist(rng), a1 = dist(rng), a2 = dist(rng);
    CoeffTensor lam0 = analyze(sample(spec, [&](double r, double z, double th) {
        return (1 - r * r) * (1 - z * z) * (a0 + a1 * r * std::cos(th)) * 0.5;
    }));
    CoeffTensor gam0 = analyze(sample(spec, [&](double r, double z, double th) {
        return (1 - r * r) * (1 - z * z) * (1 + a2 * r * std::sin(th)) * 0.25;
    }));
    const PTScalars omega0 = curl_pt(PTScalars(std::move(lam0), std::move(gam0)));
    NSConfig nc;
    nc.spec = spec;
    nc.reynolds = cfg.reynolds;
    nc.h = cfg.h;
    nc.order = cfg.bdf_order;
    nc.adi_tol = cfg.adi_tol;
    const auto t0 = std::chrono::steady_clock::now();
    NSRunResult run = ns_run(nc, omega0, cfg.steps, cfg.output_every);  // cylspec_main.cpp:200
    const double sec = seconds_since(t0);
    write_field((outdir / "omega_toroidal.ccf").string(), run.final_omega.lambda);
    write_field((outdir / "omega_poloidal.ccf").string(), run.final_omega.gamma);
    const VectorFieldCoeffs vfinal = pt_synthesize(velocity_from_vorticity(run.final_omega, cfg.adi_tol));
    Manifest mf;
    mf.put("command", jstr("ns"));
    mf.put("config", config_json(cfg));
    mf.put("timings", "{\"total_seconds\": " + jnum(sec) + ", \"per_step_seconds\": " +
                          jnum(cfg.steps ? sec / cfg.steps : 0) + "}");
    mf.put("final_time", jnum(run.final_time));
    mf.put("final_divergence", jnum(divergence(vfinal).max_abs()));
    mf.put("outputs", "[\"omega_toroidal.ccf\", \"omega_poloidal.ccf\"]");
    mf.write(outdir);
    return kExitOk;
}

int run_transform(const RunConfig& cfg) {
    if (cfg.input_path.empty()) throw ConfigError("transform requires an input FieldFile (--in)");
    const fs::path outdir(cfg.output_path);
    fs::create_directories(outdir);
    FieldVariant v = read_field(cfg.input_path);
    std::string outname;
    if (std::holds_alternative<GridField>(v)) {
        outname = "coefficients.ccf";
        write_field((outdir / outname).string(), analyze(std::get<GridField>(v)));
    } else {
        outname = "values.ccf";
        write_field((outdir / outname).string(), synthesize(std::get<CoeffTensor>(v)));
    }
    Manifest mf;
    mf.put("command", jstr("transform"));
    mf.put("config", config_json(cfg));
    mf.put("outputs", "[" + jstr(outname) + "]");
    mf.write(outdir);
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        std::cerr << "Spectral heat/Poisson/Navier-Stokes solvers in the closed cylinder (B200)\n"
                     "usage: cylspec heat|poisson|ns|bench|transform [--config F] [--m M] [--n N] [--p P] "
                     "[--steps S] [--h H] [--alpha A] [--re RE] [--bdf B] [--tol T] [--out DIR] [--in F] "
                     "[--seed S] [--case C] [--output-every K]\n";
        if (argc < 2) {
            std::cerr << "A subcommand is required\n";
            return kCliRequired;
        }
        return kExitOk;
    }
    const std::string sub = argv[1];
    if (sub != "heat" && sub != "poisson" && sub != "ns" && sub != "bench" && sub != "transform") {
        std::cerr << "The following arguments were not expected: " << sub << "\n";
        return kCliExtras;
    }
    std::map<std::string, std::string> opt;
    for (int a = 2; a < argc; ++a) {
        std::string k = argv[a];
        if (k.rfind("--", 0) != 0) {
            std::cerr << "The following arguments were not expected: " << k << "\n";
            return kCliExtras;
        }
        std::string v;
        const size_t eq = k.find('=');
        if (eq != std::string::npos) {
            v = k.substr(eq + 1);
            k = k.substr(0, eq);
        } else if (a + 1 < argc) {
            v = argv[++a];
        } else {
            std::cerr << k << " requires an argument\n";
            return kCliConversion;
        }
        static const char* known[] = {"--config", "--m", "--n", "--p", "--steps", "--h", "--alpha", "--re", "--bdf",
                                      "--tol", "--out", "--in", "--seed", "--case", "--output-every"};
        if (std::find(std::begin(known), std::end(known), k) == std::end(known)) {
            std::cerr << "The following arguments were not expected: " << k << "\n";
            return kCliExtras;
        }
        opt[k] = v;
    }
    try {
        RunConfig cfg;
        try {
            cfg = load_config(opt.count("--config") ? opt["--config"] : "");
        } catch (const ConfigError&) {
            throw;
        }
        cfg.problem = sub;
        auto toi = [&](const std::string& k, auto& dst) {
            if (!opt.count(k)) return;
            size_t end = 0;
            long long v = 0;
            try {
                v = std::stoll(opt[k], &end);
            } catch (...) {
                end = 0;
            }
            if (end != opt[k].size()) throw std::invalid_argument(k);
            dst = static_cast<std::decay_t<decltype(dst)>>(v);
        };
        auto tod = [&](const std::string& k, double& dst) {
            if (!opt.count(k)) return;
            size_t end = 0;
            try {
                dst = std::stod(opt[k], &end);
            } catch (...) {
                end = 0;
            }
            if (end != opt[k].size()) throw std::invalid_argument(k);
        };
        try {
            toi("--m", cfg.m);
            toi("--n", cfg.n);
            toi("--p", cfg.p);
            toi("--steps", cfg.steps);
            tod("--h", cfg.h);
            tod("--alpha", cfg.alpha);
            tod("--re", cfg.reynolds);
            toi("--bdf", cfg.bdf_order);
            tod("--tol", cfg.adi_tol);
            toi("--seed", cfg.seed);
            toi("--output-every", cfg.output_every);
        } catch (const std::invalid_argument& e) {
            std::cerr << "Could not convert: " << e.what() << " = " << opt[e.what()] << "\n";
            return kCliConversion;
        }
        if (opt.count("--out")) cfg.output_path = opt["--out"];
        if (opt.count("--in")) cfg.input_path = opt["--in"];
        if (opt.count("--case")) cfg.case_name = opt["--case"];
        if (const char* threads = std::getenv("CYLSPEC_THREADS")) cfg.threads = std::max(1, std::atoi(threads));
        cfg.validate();
        if (cfg.problem == "heat") return run_heat(cfg);
        if (cfg.problem == "poisson") return run_poisson(cfg);
        if (cfg.problem == "ns") return run_ns(cfg);
        if (cfg.problem == "bench")
            throw ConfigError("bench: the Table-1 method comparison (collocation / finite-difference / dense "
                              "baselines) is outside the B200 hot path; tools/heat_table1.py runs the spectral column");
        return run_transform(cfg);
    } catch (const ConfigError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return kExitConfig;
    } catch (const DomainError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return kExitConfig;
    } catch (const FieldFileError& e) {
        std::cerr << "i/o error: " << e.what() << "\n";
        return kExitNumerical;
    } catch (const std::exception& e) {
        std::cerr << "numerical failure: " << e.what() << "\n";
        try {
            fs::create_directories("out");
            std::ofstream os(fs::path("out") / "failure_manifest.json");
            os << "{\n  \"error\": " << jstr(e.what()) << "\n}\n";
        } catch (...) {
        }
        return kExitNumerical;
    }
}
