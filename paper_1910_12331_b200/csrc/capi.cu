// C ABI: include/cpkit.h (drop-in for the reference proj/include/cpkit.h,
// implemented after proj/src/capi/cpkit_c.cpp:18-389 semantics) and
// include/cpkit_dev.h (device-level seams).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <thread>

#include "../../include/cpkit.h"
#include "../../include/cpkit_dev.h"
#include "json.h"
#include "solver.h"
#include "tiny.h"
#include "selftest.h"

using cpkit::Json;

struct cpkit_tensor {
    cpkit::DenseTensor t;
};
struct cpkit_model {
    cpkit::KruskalModel m;
};
struct cpkit_instance {  // InstanceResult (report.hpp:43-48)
    cpkit::TerminalStatus status = cpkit::TerminalStatus::cap_hit;
    int iterations = 0;
    double final_residual = 1.0, best_residual = 1.0;
};
struct cpkit_report {
    std::string kind = "trace";
    Json config = Json::object();
    cpkit::ConvergenceReport trace;
    struct LikRank {  // LikelihoodRankResult (report.hpp:50-56)
        int rank = 0;
        std::vector<std::vector<cpkit_instance>> instances;
        std::vector<int> converged_inits_per_problem;
        double fraction = 0.0;
    };
    std::vector<LikRank> likelihood;
    struct Arm {  // MatmulArmResult (report.hpp:62-67)
        std::string name;
        double success_tol = 0.0;
        std::vector<cpkit_instance> inits;
        int converged = 0;
    };
    std::uint64_t matmul_n = 0;
    int matmul_rank = 0;
    std::vector<Arm> arms;
    struct BenchRow {  // report.hpp:75-81
        std::uint64_t order = 0, s = 0;
        int rank = 0, reps = 0;
        double seconds_per_matvec = 0.0;
    };
    std::vector<BenchRow> bench;
    struct Check {  // SelftestRow
        std::string name;
        int instances = 0;
        double max_rel_error = 0.0, tolerance = 0.0;
        bool pass = false;
    };
    std::vector<Check> checks;
    bool all_pass = false;
};
struct cpkit_dev_problem {
    std::unique_ptr<cpkit::Context> ctx;
    std::unique_ptr<cpkit::DeviceProblem> p;
};

namespace {

thread_local std::string g_last_error;

cpkit_status fail(cpkit_status code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

// Exceptions never cross the ABI (cpkit_c.cpp:38-62).
template <typename Fn>
cpkit_status guarded(Fn&& fn) {
    try {
        fn();
        return CPKIT_OK;
    } catch (const cpkit::InvalidArgument& e) {
        return fail(CPKIT_ERR_INVALID_ARGUMENT, e.what());
    } catch (const cpkit::ParseError& e) {
        return fail(CPKIT_ERR_PARSE, e.what());
    } catch (const cpkit::IoError& e) {
        return fail(CPKIT_ERR_IO, e.what());
    } catch (const cpkit::SingularSystem& e) {
        return fail(CPKIT_ERR_SINGULAR, e.what());
    } catch (const cpkit::NumericalFailure& e) {
        return fail(CPKIT_ERR_NUMERICAL, e.what());
    } catch (const cpkit::LimitExceeded& e) {
        return fail(CPKIT_ERR_LIMIT, e.what());
    } catch (const std::bad_alloc&) {
        return fail(CPKIT_ERR_INTERNAL, "out of host memory");
    } catch (const std::exception& e) {
        return fail(CPKIT_ERR_INTERNAL, e.what());
    } catch (...) {
        return fail(CPKIT_ERR_INTERNAL, "unknown error");
    }
}
cpkit_status require(bool ok, const char* msg) { return ok ? CPKIT_OK : fail(CPKIT_ERR_INVALID_ARGUMENT, msg); }
char* dup_string(const std::string& s) {
    char* out = new char[s.size() + 1];
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}
Json parse_config(const char* cfg) { return cfg ? Json::parse(cfg) : Json::object(); }

int current_device() {
    if (const char* e = std::getenv("CPKIT_DEVICE")) return std::atoi(e);
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) d = 0;
    return d;
}

// ---- config parsing (harness.cpp:88-167) and resolution (:203-303)
enum class InitKind { family_default, uniform, gaussian };
struct InitDist {
    InitKind kind = InitKind::family_default;
    double a = 0.0, b = 1.0;
};
struct Spec {
    std::string family = "gaussian";
    double fa = 0.0, fb = 1.0;
    std::vector<std::uint64_t> dims;
    std::vector<int> ranks{1};
    std::string optimizer = "als";
    cpkit::AlsConfig als;
    cpkit::GnConfig gn;
    int problems = 1, inits = 1;
    InitDist init;
    std::uint64_t seed = 0;
    int threads = 0;
    std::uint64_t matmul_n = 2;
};

cpkit::AlsConfig als_from_json(const Json& j) {
    cpkit::AlsConfig c;
    if (!j.contains("als")) return c;
    const Json& a = j.at("als");
    c.max_sweeps = a.value("max_sweeps", c.max_sweeps);
    c.residual_tol = a.value("residual_tol", c.residual_tol);
    c.step_tol = a.value("step_tol", c.step_tol);
    c.lambda0 = a.value("lambda0", c.lambda0);
    c.decay_factor = a.value("decay_factor", c.decay_factor);
    if (a.contains("decay_every") && !a.at("decay_every").is_null())
        c.decay_every = static_cast<int>(a.at("decay_every").as_int());
    return c;
}
cpkit::RegShape shape_from_string(const std::string& s) {
    if (s == "identity") return cpkit::RegShape::identity;
    if (s == "diagonal") return cpkit::RegShape::diagonal;
    throw cpkit::ParseError("unknown regularization shape: " + s);
}
cpkit::GnConfig gn_from_block(const Json& g) {
    cpkit::GnConfig c;
    c.grad_tol = g.value("grad_tol", c.grad_tol);
    c.residual_tol = g.value("residual_tol", c.residual_tol);
    c.step_tol = g.value("step_tol", c.step_tol);
    c.max_iters = g.value("max_iters", c.max_iters);
    c.cg_tol = g.value("cg_tol", c.cg_tol);
    c.cg_max_iters = g.value("cg_max_iters", c.cg_max_iters);
    if (g.contains("reg")) {
        const Json& r = g.at("reg");
        const std::string mode = r.value("mode", "varying");
        const cpkit::RegShape shape = shape_from_string(r.value("shape", "identity"));
        if (mode == "constant") {
            c.schedule = cpkit::RegSchedule::constant(r.value("lambda", 1e-3), shape);
        } else if (mode == "varying") {
            const double upper = r.value("upper", 1e-2);
            c.schedule = cpkit::RegSchedule::varying(upper, r.value("lower", 1e-6), r.value("mu", 2.0), shape);
            c.schedule.lambda = r.value("lambda", upper);
        } else {
            throw cpkit::ParseError("unknown regularization mode: " + mode);
        }
    }
    if (g.contains("armijo")) {
        const Json& ar = g.at("armijo");
        if (ar.is_boolean()) {
            if (ar.as_bool()) c.armijo = cpkit::ArmijoParams{};
        } else if (ar.value("enabled", true)) {
            cpkit::ArmijoParams ap;
            ap.c1 = ar.value("c1", ap.c1);
            ap.shrink = ar.value("shrink", ap.shrink);
            ap.max_backtracks = ar.value("max_backtracks", ap.max_backtracks);
            c.armijo = ap;
        }
    }
    const std::string beta = g.value("cg_beta", "standard");
    if (beta == "standard") c.cg_beta = cpkit::CgBetaVariant::standard;
    else if (beta == "stale_denominator") c.cg_beta = cpkit::CgBetaVariant::stale_denominator;
    else throw cpkit::ParseError("unknown cg_beta variant: " + beta);
    // B200 extension: "naive" = the reference's third contraction for residual_after
    const std::string ra = g.value("residual_after", "tree");
    if (ra == "naive") c.residual_naive = true;
    else if (ra != "tree") throw cpkit::ParseError("unknown residual_after mode: " + ra);
    return c;
}
cpkit::GnConfig gn_from_json(const Json& j) {
    return j.contains("gn") ? gn_from_block(j.at("gn")) : cpkit::GnConfig{};
}
InitDist init_from_json(const Json& j) {
    InitDist d;
    if (!j.contains("init")) return d;
    const Json& i = j.at("init");
    const std::string name = i.value("distribution", "default");
    if (name == "default") d.kind = InitKind::family_default;
    else if (name == "uniform") {
        d.kind = InitKind::uniform;
        d.a = i.value("a", 0.0);
        d.b = i.value("b", 1.0);
    } else if (name == "gaussian") d.kind = InitKind::gaussian;
    else throw cpkit::ParseError("unknown init distribution: " + name);
    return d;
}
void family_from_json(const Json& p, Spec& s) {
    const std::string name = p.value("family", "uniform01");
    if (name == "uniform01") { s.family = "uniform"; s.fa = 0.0; s.fb = 1.0; }
    else if (name == "uniform11") { s.family = "uniform"; s.fa = -1.0; s.fb = 1.0; }
    else if (name == "uniform") { s.family = "uniform"; s.fa = p.value("a", 0.0); s.fb = p.value("b", 1.0); }
    else if (name == "gaussian") { s.family = "gaussian"; }
    else if (name == "matmul") { s.family = "matmul"; }
    else throw cpkit::ParseError("unknown problem family: " + name);
}
int resolved_threads(int t) {
    if (t > 0) return t;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}
Spec spec_from_json(const Json& j) {  // harness.cpp:242-276
    Spec s;
    const Json problem = j.contains("problem") ? j.at("problem") : Json::object();
    family_from_json(problem, s);
    if (s.family == "matmul") {
        const std::uint64_t n = problem.value("matmul_n", 2ull);
        s.matmul_n = n;
        s.dims = {n * n, n * n, n * n};
    } else if (problem.contains("dims")) {
        s.dims.clear();
        for (const auto& d : problem.at("dims").items()) s.dims.push_back(d.as_uint());
    } else {
        throw cpkit::ParseError("experiment: problem.dims required");
    }
    if (problem.contains("ranks")) {
        s.ranks.clear();
        for (const auto& r : problem.at("ranks").items()) s.ranks.push_back(static_cast<int>(r.as_int()));
    } else if (problem.contains("rank")) {
        s.ranks = {static_cast<int>(problem.at("rank").as_int())};
    }
    s.optimizer = j.value("optimizer", "als");
    if (s.optimizer != "als" && s.optimizer != "gn") throw cpkit::ParseError("unknown optimizer: " + s.optimizer);
    s.als = als_from_json(j);
    s.gn = gn_from_json(j);
    s.problems = j.value("problems", 1);
    s.inits = j.value("inits", 1);
    s.init = init_from_json(j);
    s.seed = j.value("seed", 0ull);
    s.threads = j.value("threads", 0);
    // validate (harness.cpp:203-220)
    if (s.ranks.empty()) throw cpkit::InvalidArgument("experiment: at least one rank required");
    for (int r : s.ranks)
        if (r < 1) throw cpkit::InvalidArgument("experiment: ranks must be positive");
    if (s.problems < 1 || s.inits < 1) throw cpkit::InvalidArgument("experiment: problems and inits must be >= 1");
    if (s.init.kind == InitKind::uniform && !(s.init.a < s.init.b))
        throw cpkit::InvalidArgument("experiment: init uniform needs a < b");
    if (s.family == "uniform" && !(s.fa < s.fb)) throw cpkit::InvalidArgument("problem spec: uniform needs a < b");
    if (s.dims.empty()) throw cpkit::InvalidArgument("problem spec: dims must be nonempty");
    s.als.validate();
    s.gn.validate();
    return s;
}
InitDist resolved_init(const Spec& s) {
    if (s.init.kind != InitKind::family_default) return s.init;
    InitDist d;
    if (s.family == "uniform" && s.fa >= 0.0) {
        d.kind = InitKind::uniform;
        return d;
    }
    d.kind = InitKind::gaussian;
    return d;
}
Json als_to_json(const cpkit::AlsConfig& c) {
    Json a = Json::object();
    a["max_sweeps"] = c.max_sweeps;
    a["residual_tol"] = c.residual_tol;
    a["step_tol"] = c.step_tol;
    a["lambda0"] = c.lambda0;
    a["decay_factor"] = c.decay_factor;
    a["decay_every"] = c.decay_every ? Json(*c.decay_every) : Json();
    return a;
}
Json gn_to_json(const cpkit::GnConfig& c) {
    Json g = Json::object();
    g["grad_tol"] = c.grad_tol;
    g["residual_tol"] = c.residual_tol;
    g["step_tol"] = c.step_tol;
    g["max_iters"] = c.max_iters;
    g["cg_tol"] = c.cg_tol;
    g["cg_max_iters"] = c.cg_max_iters;
    Json r = Json::object();
    r["mode"] = c.schedule.mode == cpkit::RegMode::constant ? "constant" : "varying";
    r["shape"] = c.schedule.shape == cpkit::RegShape::identity ? "identity" : "diagonal";
    r["lambda"] = c.schedule.lambda;
    if (c.schedule.mode == cpkit::RegMode::varying) {
        r["mu"] = c.schedule.mu;
        r["lower"] = c.schedule.lower;
        r["upper"] = c.schedule.upper;
    }
    g["reg"] = r;
    Json a = Json::object();
    a["enabled"] = static_cast<bool>(c.armijo);
    if (c.armijo) {
        a["c1"] = c.armijo->c1;
        a["shrink"] = c.armijo->shrink;
        a["max_backtracks"] = c.armijo->max_backtracks;
    }
    g["armijo"] = a;
    g["cg_beta"] = c.cg_beta == cpkit::CgBetaVariant::standard ? "standard" : "stale_denominator";
    if (c.residual_naive) g["residual_after"] = "naive";  // only when set: the reference schema otherwise
    return g;
}
Json init_to_json(const InitDist& d) {
    Json i = Json::object();
    switch (d.kind) {
        case InitKind::family_default: i["distribution"] = "default"; break;
        case InitKind::uniform:
            i["distribution"] = "uniform";
            i["a"] = d.a;
            i["b"] = d.b;
            break;
        case InitKind::gaussian: i["distribution"] = "gaussian"; break;
    }
    return i;
}
Json resolved_json(const Spec& s) {
    Json j = Json::object();
    Json p = Json::object();
    if (s.family == "uniform") {
        p["family"] = "uniform";
        p["a"] = s.fa;
        p["b"] = s.fb;
    } else {
        p["family"] = s.family;
        if (s.family == "matmul") p["matmul_n"] = static_cast<unsigned long long>(s.matmul_n);
    }
    Json dims = Json::array();
    for (auto d : s.dims) dims.push_back(Json(static_cast<unsigned long long>(d)));
    p["dims"] = dims;
    Json ranks = Json::array();
    for (int r : s.ranks) ranks.push_back(Json(r));
    p["ranks"] = ranks;
    j["problem"] = p;
    j["optimizer"] = s.optimizer;
    j["als"] = als_to_json(s.als);
    j["gn"] = gn_to_json(s.gn);
    j["problems"] = s.problems;
    j["inits"] = s.inits;
    j["init"] = init_to_json(resolved_init(s));
    j["seed"] = static_cast<unsigned long long>(s.seed);
    j["threads"] = resolved_threads(s.threads);
    return j;
}

Json instance_to_json(const cpkit_instance& r) {  // report.cpp:56-61
    Json o = Json::object();
    o["status"] = cpkit::to_string(r.status);
    o["iterations"] = r.iterations;
    o["final_residual"] = r.final_residual;
    o["best_residual"] = r.best_residual;
    return o;
}
Json report_to_json(const cpkit_report& r) {  // report.cpp:95-141
    Json j = Json::object();
    j["kind"] = r.kind;
    j["config"] = r.config;
    if (r.kind == "likelihood") {
        Json ranks = Json::array();
        for (const auto& rr : r.likelihood) {
            Json problems = Json::array();
            for (std::size_t p = 0; p < rr.instances.size(); ++p) {
                Json inits = Json::array();
                for (const auto& inst : rr.instances[p]) inits.push_back(instance_to_json(inst));
                Json pj = Json::object();
                pj["problem"] = static_cast<unsigned long long>(p);
                pj["converged_inits"] = rr.converged_inits_per_problem[p];
                pj["inits"] = inits;
                problems.push_back(pj);
            }
            Json rj = Json::object();
            rj["rank"] = rr.rank;
            rj["fraction"] = rr.fraction;
            rj["problems"] = problems;
            ranks.push_back(rj);
        }
        j["ranks"] = ranks;
        return j;
    }
    if (r.kind == "matmul") {
        j["n"] = static_cast<unsigned long long>(r.matmul_n);
        j["rank"] = r.matmul_rank;
        Json arms = Json::array();
        for (const auto& arm : r.arms) {
            Json inits = Json::array();
            for (const auto& inst : arm.inits) inits.push_back(instance_to_json(inst));
            Json aj = Json::object();
            aj["name"] = arm.name;
            aj["success_tol"] = arm.success_tol;
            aj["converged"] = arm.converged;
            aj["inits"] = inits;
            arms.push_back(aj);
        }
        j["arms"] = arms;
        return j;
    }
    if (r.kind == "bench") {
        Json rows = Json::array();
        for (const auto& b : r.bench) {
            Json o = Json::object();
            o["order"] = static_cast<unsigned long long>(b.order);
            o["s"] = static_cast<unsigned long long>(b.s);
            o["rank"] = b.rank;
            o["reps"] = b.reps;
            o["seconds_per_matvec"] = b.seconds_per_matvec;
            rows.push_back(o);
        }
        j["rows"] = rows;
        return j;
    }
    if (r.kind == "selftest") {
        Json checks = Json::array();
        for (const auto& c : r.checks) {
            Json o = Json::object();
            o["name"] = c.name;
            o["instances"] = c.instances;
            o["max_rel_error"] = c.max_rel_error;
            o["tolerance"] = c.tolerance;
            o["pass"] = c.pass;
            checks.push_back(o);
        }
        j["checks"] = checks;
        j["all_pass"] = r.all_pass;
        return j;
    }
    j["status"] = cpkit::to_string(r.trace.status);
    Json recs = Json::array();
    for (const auto& rec : r.trace.records) {
        Json o = Json::object();
        o["iter"] = rec.iteration;
        o["residual"] = rec.residual;
        o["fitness"] = rec.fitness;
        o["lambda"] = rec.lambda;
        o["cg_iters"] = rec.cg_iters;
        o["seconds"] = rec.seconds;
        recs.push_back(o);
    }
    j["records"] = recs;
    return j;
}
std::string fmt_double(double v) { return Json(v).dump(); }
std::string report_to_csv(const cpkit_report& r) {  // report.cpp:254-300
    std::ostringstream os;
    if (r.kind == "likelihood") {
        os << "rank,problem,init,status,iterations,final_residual,best_residual\n";
        for (const auto& rr : r.likelihood)
            for (std::size_t p = 0; p < rr.instances.size(); ++p)
                for (std::size_t i = 0; i < rr.instances[p].size(); ++i) {
                    const auto& inst = rr.instances[p][i];
                    os << rr.rank << ',' << p << ',' << i << ',' << cpkit::to_string(inst.status) << ','
                       << inst.iterations << ',' << fmt_double(inst.final_residual) << ','
                       << fmt_double(inst.best_residual) << '\n';
                }
        return os.str();
    }
    if (r.kind == "matmul") {
        os << "arm,init,status,iterations,final_residual,best_residual\n";
        for (const auto& arm : r.arms)
            for (std::size_t i = 0; i < arm.inits.size(); ++i) {
                const auto& inst = arm.inits[i];
                os << arm.name << ',' << i << ',' << cpkit::to_string(inst.status) << ',' << inst.iterations << ','
                   << fmt_double(inst.final_residual) << ',' << fmt_double(inst.best_residual) << '\n';
            }
        return os.str();
    }
    if (r.kind == "bench") {
        os << "order,s,rank,reps,seconds_per_matvec\n";
        for (const auto& b : r.bench)
            os << b.order << ',' << b.s << ',' << b.rank << ',' << b.reps << ',' << fmt_double(b.seconds_per_matvec)
               << '\n';
        return os.str();
    }
    if (r.kind == "selftest") {
        os << "check,instances,max_rel_error,tolerance,pass\n";
        for (const auto& c : r.checks)
            os << c.name << ',' << c.instances << ',' << fmt_double(c.max_rel_error) << ','
               << fmt_double(c.tolerance) << ',' << (c.pass ? 1 : 0) << '\n';
        return os.str();
    }
    os << "iter,residual,fitness,lambda,cg_iters,seconds\n";
    for (const auto& rec : r.trace.records)
        os << rec.iteration << ',' << fmt_double(rec.residual) << ',' << fmt_double(rec.fitness) << ','
           << fmt_double(rec.lambda) << ',' << rec.cg_iters << ',' << fmt_double(rec.seconds) << '\n';
    return os.str();
}

cpkit::KruskalModel start_model(const std::vector<std::uint64_t>& dims, const Json& j, const Spec& spec) {
    const int rank = j.value("rank", 0);
    if (rank < 1) throw cpkit::InvalidArgument("cpkit_decompose: rank required when init is null");
    InitDist dist = spec.init;
    if (dist.kind == InitKind::family_default) dist.kind = InitKind::gaussian;
    const std::uint64_t seed = cpkit::init_seed(spec.seed, rank, 0, 0);
    return dist.kind == InitKind::uniform ? cpkit::random_model_uniform(dims, rank, seed, dist.a, dist.b)
                                          : cpkit::random_model_gaussian(dims, rank, seed);
}

// Runs the selected optimizer on a device problem; fills model + report.
void run_optimizer(cpkit::DeviceProblem& p, const std::string& optimizer, const Spec& spec,
                   cpkit::KruskalModel start, cpkit::KruskalModel& result, cpkit_report& report) {
    if (optimizer == "als") {
        auto [m, rep] = cpkit::als_optimize(p, std::move(start), spec.als);
        result = std::move(m);
        report.trace = std::move(rep);
    } else if (optimizer == "gn") {
        auto [m, rep] = cpkit::gn_optimize(p, std::move(start), spec.gn);
        result = std::move(m);
        report.trace = std::move(rep);
    } else {
        throw cpkit::ParseError("cpkit_decompose: unknown optimizer " + optimizer);
    }
}

cpkit::KruskalModel model_from_stacked(const std::vector<std::uint64_t>& dims, std::int64_t rank,
                                       const double* buf) {
    cpkit::KruskalModel m;
    m.dims = dims;
    m.rank = rank;
    std::size_t at = 0;
    for (auto d : dims) {
        cpkit::Matrix a(static_cast<std::int64_t>(d), rank);
        std::memcpy(a.data.data(), buf + at, a.data.size() * 8);
        at += a.data.size();
        m.factors.push_back(std::move(a));
    }
    return m;
}
void model_to_stacked(const cpkit::KruskalModel& m, double* buf) {
    std::size_t at = 0;
    for (const auto& a : m.factors) {
        std::memcpy(buf + at, a.data.data(), a.data.size() * 8);
        at += a.data.size();
    }
}

// ---- batched independent instances (harness.cpp:433-459, :488-653) ----------------------
// Tensor entries in the reference's per-entry order (kruskal.cpp:76-90).
std::vector<double> reconstruct_host(const cpkit::KruskalModel& m) {
    const int N = static_cast<int>(m.dims.size());
    std::uint64_t total = 1;
    for (auto d : m.dims) total *= d;
    std::vector<double> out(total);
    std::vector<std::uint64_t> idx(N);
    for (std::uint64_t f = 0; f < total; ++f) {
        std::uint64_t rem = f;
        for (int n = N - 1; n >= 0; --n) {
            idx[n] = rem % m.dims[n];
            rem /= m.dims[n];
        }
        double acc = 0.0;
        for (std::int64_t r = 0; r < m.rank; ++r) {
            double prod = 1.0;
            for (int n = 0; n < N; ++n) {
                const double v = m.factors[n].data[idx[n] * m.rank + r];
                prod = prod * v;
            }
            acc = acc + prod;
        }
        out[f] = acc;
    }
    return out;
}
// matmul_tensor (generators.cpp:96-117): T[i n + j, i n + l, l n + j] = 1
std::vector<double> matmul_data(std::uint64_t n) {
    const std::uint64_t sq = n * n;
    std::vector<double> t(sq * sq * sq, 0.0);
    for (std::uint64_t i = 0; i < n; ++i)
        for (std::uint64_t l = 0; l < n; ++l)
            for (std::uint64_t jj = 0; jj < n; ++jj) t[((i * n + jj) * sq + i * n + l) * sq + l * n + jj] = 1.0;
    return t;
}

struct BatchJob {
    std::vector<std::uint64_t> dims;
    int rank = 1;
    bool gn = false;
    cpkit::AlsConfig als;
    cpkit::GnConfig gncfg;
    std::vector<std::vector<double>> tensors;  // distinct problem tensors
    std::vector<int> x_index;                  // instance -> tensor
    std::vector<cpkit::KruskalModel> inits;    // instance starts
};
cpkit::TerminalStatus status_of(int s) {
    switch (s) {
        case 0: return cpkit::TerminalStatus::converged_residual;
        case 1: return cpkit::TerminalStatus::converged_step;
        case 2: return cpkit::TerminalStatus::cap_hit;
        default: return cpkit::TerminalStatus::numerical_failure;
    }
}
cpkit_instance summarize(const cpkit::ConvergenceReport& rep) {  // harness.cpp:433-441
    cpkit_instance r;
    r.status = rep.status;
    r.iterations = static_cast<int>(rep.records.size());
    r.final_residual = rep.final_residual();
    r.best_residual = rep.best_residual();
    return r;
}

// One CTA per instance (kernels_tiny.cu): device buffers of a launched batch.
struct TinyRun {
    int count = 0, S = 0;
    bool want_factors = false;
    cpkit::DevBuf<double> dx, da, dl, dfac, dfin, dbest;
    cpkit::DevBuf<int> dxi, dst, dit;
};
// Launches the job's batch on `st` (asynchronously); nullptr when the shape
// does not fit one CTA (or CPKIT_NO_TINY is set).
std::unique_ptr<TinyRun> tiny_launch(const BatchJob& job, bool want_factors, cudaStream_t st) {
    const int count = static_cast<int>(job.inits.size());
    cpkit::TinyLayout lay{};
    int numel = 0, S = 0;
    const int N = static_cast<int>(job.dims.size());
    if (count == 0 || !cpkit::tiny_layout(N, job.dims.data(), job.rank, lay, numel, S) || std::getenv("CPKIT_NO_TINY"))
        return nullptr;
    auto run = std::make_unique<TinyRun>();
    run->count = count;
    run->S = S;
    run->want_factors = want_factors;
    cpkit::TinyParams tp{};
    tp.order = N;
    tp.rank = job.rank;
    tp.off[0] = 0;
    for (int n = 0; n < N; ++n) {
        tp.dims[n] = static_cast<int>(job.dims[n]);
        tp.off[n + 1] = tp.off[n] + tp.dims[n] * job.rank;
    }
    tp.S = S;
    tp.numel = numel;
    tp.count = count;
    tp.optimizer = job.gn ? 1 : 0;
    // ALS is a chain of small serial solves (one warp: cheapest barriers); GN's
    // matvec passes parallelise over the stacked entries (measured: ALS 32, GN 128)
    tp.threads = (!job.gn && S <= 256 && job.rank <= 16 && numel <= 1024) ? 32 : cpkit::kTinyThreads;
    if (const char* e = std::getenv("CPKIT_TINY_THREADS")) tp.threads = std::max(32, std::min(cpkit::kTinyThreads, std::atoi(e)));
    tp.layout = lay;
    std::vector<double> lambdas;
    {
        const auto& a = job.als;
        tp.als.max_sweeps = a.max_sweeps;
        tp.als.residual_tol = a.residual_tol;
        tp.als.step_tol = a.step_tol;
        tp.als.lambda0 = a.lambda0;
        tp.als.decay_every = a.decay_every ? *a.decay_every : 0;
        if (tp.als.decay_every > 0) {  // lambda_k = lambda0 / decay^k (als.cpp:66-67, host std::pow)
            const int nk = a.max_sweeps / tp.als.decay_every + 1;
            for (int k = 0; k < nk; ++k) lambdas.push_back(a.lambda0 / std::pow(a.decay_factor, static_cast<double>(k)));
        }
    }
    {
        const auto& g = job.gncfg;
        tp.gn.grad_tol = g.grad_tol;
        tp.gn.residual_tol = g.residual_tol;
        tp.gn.step_tol = g.step_tol;
        tp.gn.cg_tol = g.cg_tol;
        tp.gn.max_iters = g.max_iters;
        std::uint64_t total = 0;
        for (auto d : job.dims) total += d * static_cast<std::uint64_t>(job.rank);
        tp.gn.cap = g.cg_max_iters > 0 ? g.cg_max_iters
                                       : static_cast<int>(std::min<std::uint64_t>(total, 10ull * job.rank));
        tp.gn.mode = g.schedule.mode == cpkit::RegMode::varying ? 1 : 0;
        tp.gn.shape = g.schedule.shape == cpkit::RegShape::diagonal ? 1 : 0;
        tp.gn.lambda = g.schedule.lambda;
        tp.gn.mu = g.schedule.mu;
        tp.gn.lower = g.schedule.lower;
        tp.gn.upper = g.schedule.upper;
        tp.gn.direction = g.schedule.direction == cpkit::RegSchedule::Direction::up ? 1 : 0;
        tp.gn.armijo = g.armijo ? 1 : 0;
        const cpkit::ArmijoParams ap = g.armijo ? *g.armijo : cpkit::ArmijoParams{};
        tp.gn.c1 = ap.c1;
        tp.gn.shrink = ap.shrink;
        tp.gn.max_backtracks = ap.max_backtracks;
        tp.gn.beta_variant = g.cg_beta == cpkit::CgBetaVariant::stale_denominator ? 1 : 0;
    }
    std::vector<double> xs;
    for (const auto& t : job.tensors) xs.insert(xs.end(), t.begin(), t.end());
    std::vector<double> a0(static_cast<std::size_t>(count) * S);
    for (int i = 0; i < count; ++i) model_to_stacked(job.inits[i], a0.data() + static_cast<std::size_t>(i) * S);
    run->dx.resize(xs.size());
    run->da.resize(a0.size());
    run->dl.resize(std::max<std::size_t>(1, lambdas.size()));
    run->dfac.resize(want_factors ? a0.size() : 1);
    run->dfin.resize(count);
    run->dbest.resize(count);
    run->dxi.resize(count);
    run->dst.resize(count);
    run->dit.resize(count);
    CPK_CUDA(cudaMemcpy(run->dx.get(), xs.data(), xs.size() * 8, cudaMemcpyHostToDevice));
    CPK_CUDA(cudaMemcpy(run->da.get(), a0.data(), a0.size() * 8, cudaMemcpyHostToDevice));
    if (!lambdas.empty())
        CPK_CUDA(cudaMemcpy(run->dl.get(), lambdas.data(), lambdas.size() * 8, cudaMemcpyHostToDevice));
    CPK_CUDA(cudaMemcpy(run->dxi.get(), job.x_index.data(), count * sizeof(int), cudaMemcpyHostToDevice));
    tp.als.lambdas = run->dl.get();
    tp.x = run->dx.get();
    tp.x_index = run->dxi.get();
    tp.init = run->da.get();
    tp.factors_out = want_factors ? run->dfac.get() : nullptr;
    tp.status = run->dst.get();
    tp.iterations = run->dit.get();
    tp.final_residual = run->dfin.get();
    tp.best_residual = run->dbest.get();
    cpkit::launch_tiny(tp, st);
    return run;
}
// After the launch stream has drained: per-instance results (and factors).
std::vector<cpkit_instance> tiny_collect(TinyRun& run, std::vector<std::vector<double>>* factors) {
    const int count = run.count;
    std::vector<int> st(count), it(count);
    std::vector<double> fin(count), best(count);
    CPK_CUDA(cudaMemcpy(st.data(), run.dst.get(), count * sizeof(int), cudaMemcpyDeviceToHost));
    CPK_CUDA(cudaMemcpy(it.data(), run.dit.get(), count * sizeof(int), cudaMemcpyDeviceToHost));
    CPK_CUDA(cudaMemcpy(fin.data(), run.dfin.get(), count * 8, cudaMemcpyDeviceToHost));
    CPK_CUDA(cudaMemcpy(best.data(), run.dbest.get(), count * 8, cudaMemcpyDeviceToHost));
    std::vector<cpkit_instance> out(count);
    for (int i = 0; i < count; ++i) out[i] = {status_of(st[i]), it[i], fin[i], best[i]};
    if (factors && run.want_factors) {
        std::vector<double> f(static_cast<std::size_t>(count) * run.S);
        CPK_CUDA(cudaMemcpy(f.data(), run.dfac.get(), f.size() * 8, cudaMemcpyDeviceToHost));
        factors->assign(count, {});
        for (int i = 0; i < count; ++i)
            (*factors)[i].assign(f.begin() + static_cast<std::ptrdiff_t>(i) * run.S,
                                 f.begin() + static_cast<std::ptrdiff_t>(i + 1) * run.S);
    }
    return out;
}

// Runs every instance of the job: one CTA per instance (kernels_tiny.cu) when
// the shape fits a CTA, else one device problem per instance. factors (when
// non-null) receives each instance's final stacked factors.
std::vector<cpkit_instance> run_batch(const BatchJob& job, std::vector<std::vector<double>>* factors) {
    const int count = static_cast<int>(job.inits.size());
    std::vector<cpkit_instance> out(count);
    if (count == 0) return out;
    if (job.gn) job.gncfg.validate();
    else job.als.validate();
    int S = 0;
    for (auto d : job.dims) S += static_cast<int>(d) * job.rank;
    if (auto run = tiny_launch(job, factors != nullptr, 0)) {
        CPK_CUDA(cudaDeviceSynchronize());
        return tiny_collect(*run, factors);
    }
    // larger instances: one device problem per tensor, instances in sequence
    cpkit::Context ctx(current_device());
    if (factors) factors->assign(count, {});
    for (std::size_t t = 0; t < job.tensors.size(); ++t) {
        cpkit::DeviceProblem p(ctx, job.dims, job.rank);
        p.upload_tensor(job.tensors[t].data());
        for (int i = 0; i < count; ++i) {
            if (job.x_index[i] != static_cast<int>(t)) continue;
            cpkit::KruskalModel result = job.inits[i];
            try {  // run_instance (harness.cpp:443-459)
                // fault injection for the boundary tests only: a device failure
                // inside an instance must surface as CPKIT_ERR_INTERNAL
                if (std::getenv("CPKIT_INJECT_DEVICE_FAULT")) throw cpkit::DeviceError("injected device fault");
                if (job.gn) {
                    auto [m, rep] = cpkit::gn_optimize(p, job.inits[i], job.gncfg);
                    out[i] = summarize(rep);
                    result = std::move(m);
                } else {
                    auto [m, rep] = cpkit::als_optimize(p, job.inits[i], job.als);
                    out[i] = summarize(rep);
                    result = std::move(m);
                }
            } catch (const cpkit::DeviceError&) {
                throw;  // a CUDA fault leaves the context unusable: CPKIT_ERR_INTERNAL
            } catch (const cpkit::Error&) {
                out[i] = cpkit_instance{};
                out[i].status = cpkit::TerminalStatus::numerical_failure;
            }
            if (factors) {
                (*factors)[i].resize(static_cast<std::size_t>(S));
                model_to_stacked(result, (*factors)[i].data());
            }
        }
    }
    return out;
}

struct EventPair {
    cudaEvent_t a{}, b{};
    EventPair() {
        CPK_CUDA(cudaEventCreate(&a));
        CPK_CUDA(cudaEventCreate(&b));
    }
    ~EventPair() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    float ms() {
        CPK_CUDA(cudaEventSynchronize(b));
        float v = 0;
        CPK_CUDA(cudaEventElapsedTime(&v, a, b));
        return v;
    }
};

}  // namespace

extern "C" {

const char* cpkit_version(void) { return "1.0.0"; }

const char* cpkit_status_name(cpkit_status status) {
    switch (status) {
        case CPKIT_OK: return "ok";
        case CPKIT_ERR_INVALID_ARGUMENT: return "invalid_argument";
        case CPKIT_ERR_PARSE: return "parse_error";
        case CPKIT_ERR_IO: return "io_error";
        case CPKIT_ERR_SINGULAR: return "singular_system";
        case CPKIT_ERR_NUMERICAL: return "numerical_failure";
        case CPKIT_ERR_LIMIT: return "limit_exceeded";
        case CPKIT_ERR_INTERNAL: return "internal_error";
    }
    return "unknown";
}
const char* cpkit_last_error(void) { return g_last_error.c_str(); }
void cpkit_string_free(char* s) { delete[] s; }

// ---- tensors -------------------------------------------------------------------
cpkit_status cpkit_tensor_create(const uint64_t* dims, uint64_t order, const double* data, cpkit_tensor** out) {
    if (auto st = require(dims && data && out && order > 0, "cpkit_tensor_create: null argument")) return st;
    return guarded([&] {
        std::vector<std::uint64_t> d(dims, dims + order);
        const std::uint64_t total = cpkit::product_of_dims(d);
        std::vector<double> v(data, data + total);
        auto t = cpkit::DenseTensor::from_data(std::move(d), std::move(v));
        t.validate();
        *out = new cpkit_tensor{std::move(t)};
    });
}
cpkit_status cpkit_tensor_load(const char* path, cpkit_tensor** out) {
    if (auto st = require(path && out, "cpkit_tensor_load: null argument")) return st;
    return guarded([&] { *out = new cpkit_tensor{cpkit::read_tensor(path)}; });
}
cpkit_status cpkit_tensor_save(const cpkit_tensor* t, const char* path) {
    if (auto st = require(t && path, "cpkit_tensor_save: null argument")) return st;
    return guarded([&] { cpkit::write_tensor(t->t, path); });
}
uint64_t cpkit_tensor_order(const cpkit_tensor* t) { return t ? t->t.order() : 0; }
uint64_t cpkit_tensor_extent(const cpkit_tensor* t, uint64_t mode) {
    return (t && mode < t->t.order()) ? t->t.extent(mode) : 0;
}
uint64_t cpkit_tensor_element_count(const cpkit_tensor* t) { return t ? t->t.size() : 0; }
const double* cpkit_tensor_data(const cpkit_tensor* t) { return t ? t->t.data() : nullptr; }
void cpkit_tensor_destroy(cpkit_tensor* t) { delete t; }

// ---- models ----------------------------------------------------------------------
cpkit_status cpkit_model_load(const char* path, cpkit_model** out) {
    if (auto st = require(path && out, "cpkit_model_load: null argument")) return st;
    return guarded([&] { *out = new cpkit_model{cpkit::read_model(path)}; });
}
cpkit_status cpkit_model_save(const cpkit_model* m, const char* path) {
    if (auto st = require(m && path, "cpkit_model_save: null argument")) return st;
    return guarded([&] { cpkit::write_model(m->m, path); });
}
uint64_t cpkit_model_order(const cpkit_model* m) { return m ? m->m.order() : 0; }
uint64_t cpkit_model_rank(const cpkit_model* m) { return m ? static_cast<uint64_t>(m->m.rank) : 0; }
uint64_t cpkit_model_extent(const cpkit_model* m, uint64_t mode) {
    return (m && mode < m->m.order()) ? m->m.dims[mode] : 0;
}
const double* cpkit_model_factor(const cpkit_model* m, uint64_t mode) {
    return (m && mode < m->m.order()) ? m->m.factors[mode].data.data() : nullptr;
}
namespace {
cpkit::DenseTensor reconstruct_on_device(const cpkit::KruskalModel& m, std::uint64_t cap) {
    m.validate();
    const std::uint64_t total = cpkit::product_of_dims(m.dims);
    if (total > cap) throw cpkit::LimitExceeded("reconstruct: element count exceeds cap");
    cpkit::DenseTensor t(m.dims);
    if (m.order() < 2) {  // order-1 model: the single factor's row sums
        for (std::uint64_t i = 0; i < total; ++i) {
            double acc = 0.0;
            for (std::int64_t r = 0; r < m.rank; ++r) acc += m.factors[0].data[i * m.rank + r];
            t.data()[i] = acc;
        }
        return t;
    }
    cpkit::Context ctx(current_device());
    cpkit::DeviceProblem p(ctx, m.dims, static_cast<int>(m.rank));
    p.generate_tensor(m, 0, 0.0);
    p.download_tensor(t.data());
    return t;
}
}  // namespace
cpkit_status cpkit_model_reconstruct(const cpkit_model* m, cpkit_tensor** out) {
    if (auto st = require(m && out, "cpkit_model_reconstruct: null argument")) return st;
    return guarded([&] { *out = new cpkit_tensor{reconstruct_on_device(m->m, cpkit::kDefaultElementCap)}; });
}
void cpkit_model_destroy(cpkit_model* m) { delete m; }

// ---- generators (cpkit_c.cpp:198-225; generators.cpp:78-117) ---------------------
cpkit_status cpkit_generate_low_rank(const char* spec_json, cpkit_model** out_model, cpkit_tensor** out_tensor) {
    if (auto st = require(spec_json && (out_model || out_tensor), "cpkit_generate_low_rank: null argument"))
        return st;
    return guarded([&] {
        const Json j = Json::parse(spec_json);
        Json wrapped = Json::object();
        wrapped["problem"] = j;
        const Spec s = spec_from_json(wrapped);
        if (s.family == "matmul") throw cpkit::InvalidArgument("random_low_rank: family must be uniform or gaussian");
        if (cpkit::product_of_dims(s.dims) > cpkit::kDefaultElementCap)
            throw cpkit::LimitExceeded("random_low_rank: element count exceeds cap");
        const std::uint64_t seed = j.value("seed", 0ull);
        cpkit::KruskalModel model = s.family == "uniform"
                                        ? cpkit::random_model_uniform(s.dims, s.ranks[0], seed, s.fa, s.fb)
                                        : cpkit::random_model_gaussian(s.dims, s.ranks[0], seed);
        if (out_tensor) *out_tensor = new cpkit_tensor{reconstruct_on_device(model, cpkit::kDefaultElementCap)};
        if (out_model) *out_model = new cpkit_model{std::move(model)};
    });
}
cpkit_status cpkit_matmul_tensor(uint64_t n, cpkit_tensor** out) {
    if (auto st = require(out != nullptr, "cpkit_matmul_tensor: null argument")) return st;
    return guarded([&] {
        if (n < 1) throw cpkit::InvalidArgument("matmul_tensor: n must be >= 1");
        const std::uint64_t sq = n * n;
        if (sq * sq * sq > cpkit::kDefaultElementCap) throw cpkit::LimitExceeded("matmul_tensor: element count exceeds cap");
        cpkit::DenseTensor t({sq, sq, sq});
        for (std::uint64_t i = 0; i < n; ++i)
            for (std::uint64_t l = 0; l < n; ++l)
                for (std::uint64_t jj = 0; jj < n; ++jj) {
                    const std::uint64_t m0 = i * n + jj, m1 = i * n + l, m2 = l * n + jj;
                    t.data()[(m0 * sq + m1) * sq + m2] = 1.0;
                }
        *out = new cpkit_tensor{std::move(t)};
    });
}

// ---- decomposition (cpkit_c.cpp:229-297) ----------------------------------------------
cpkit_status cpkit_decompose(const cpkit_tensor* t, const char* config_json, const cpkit_model* init,
                             cpkit_model** out_model, cpkit_report** out_report) {
    if (auto st = require(t != nullptr, "cpkit_decompose: null tensor")) return st;
    return guarded([&] {
        const Json j = parse_config(config_json);
        const std::string optimizer = j.value("optimizer", "als");
        Json wrapped = j;
        Json prob = Json::object();
        prob["family"] = "gaussian";
        Json dims = Json::array();
        for (auto d : t->t.dims()) dims.push_back(Json(static_cast<unsigned long long>(d)));
        prob["dims"] = dims;
        prob["rank"] = j.value("rank", 1);
        wrapped["problem"] = prob;
        const Spec spec = spec_from_json(wrapped);

        cpkit::KruskalModel start;
        if (init != nullptr) {
            start = init->m;
            if (start.dims != t->t.dims())
                throw cpkit::InvalidArgument("cpkit_decompose: init model extents do not match tensor");
        } else {
            start = start_model(t->t.dims(), j, spec);
        }
        if (t->t.order() < 2) throw cpkit::InvalidArgument("mttkrp: tensor order must be at least 2");

        auto report = std::make_unique<cpkit_report>();
        Json cfg = resolved_json(spec);
        cfg["kind"] = "decompose";
        cfg["optimizer"] = optimizer;
        report->config = cfg;

        static const bool phase_trace = std::getenv("CPKIT_PHASE_TRACE") != nullptr;  // timing experiments
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto t0 = now();
        auto t1 = t0, t2 = t0, t3 = t0;
        {
            cpkit::Context ctx(current_device());
            cpkit::DeviceProblem p(ctx, t->t.dims(), static_cast<int>(start.rank));
            p.upload_tensor(t->t.data(), &start);  // the first back root beside the upload (orders >= 4)
            if (phase_trace) {
                ctx.sync();
                t1 = now();
            }
            cpkit::KruskalModel result;
            run_optimizer(p, optimizer, spec, std::move(start), result, *report);
            t2 = now();
            if (out_model) *out_model = new cpkit_model{std::move(result)};
            if (out_report) *out_report = report.release();
        }
        t3 = now();
        if (phase_trace)
            std::fprintf(stderr, "cpkit_decompose: setup+upload %.1f ms, optimize %.1f ms, teardown %.1f ms\n",
                         ms(t0, t1), ms(t1, t2), ms(t2, t3));
    });
}

// ---- runners ---------------------------------------------------------------------------
// run_trace (harness.cpp:461-486): one problem from the spec's family, one init.
cpkit_status cpkit_run_trace(const char* config_json, cpkit_report** out) {
    if (auto st = require(config_json && out, "cpkit_run_trace: null argument")) return st;
    return guarded([&] {
        const Spec spec = spec_from_json(Json::parse(config_json));
        const int rank = spec.ranks[0];
        const std::uint64_t ps = cpkit::problem_seed(spec.seed, rank, 0);
        const InitDist d = resolved_init(spec);
        const std::uint64_t is = cpkit::init_seed(spec.seed, rank, 0, 0);
        cpkit::KruskalModel start = d.kind == InitKind::uniform ? cpkit::random_model_uniform(spec.dims, rank, is, d.a, d.b)
                                                                : cpkit::random_model_gaussian(spec.dims, rank, is);
        auto report = std::make_unique<cpkit_report>();
        Json cfg = resolved_json(spec);
        cfg["kind"] = "trace";
        report->config = cfg;
        cpkit::Context ctx(current_device());
        cpkit::DeviceProblem p(ctx, spec.dims, rank);
        if (spec.family == "matmul") {  // build_problem_tensor (harness.cpp:422-431)
            p.upload_tensor(matmul_data(spec.matmul_n).data());
        } else {
            const cpkit::KruskalModel truth = spec.family == "uniform"
                                                  ? cpkit::random_model_uniform(spec.dims, rank, ps, spec.fa, spec.fb)
                                                  : cpkit::random_model_gaussian(spec.dims, rank, ps);
            p.generate_tensor(truth, 0, 0.0);
        }
        cpkit::KruskalModel result;
        try {
            run_optimizer(p, spec.optimizer, spec, std::move(start), result, *report);
        } catch (const cpkit::DeviceError&) {
            throw;  // CUDA fault: CPKIT_ERR_INTERNAL, not a numerical failure
        } catch (const cpkit::Error&) {
            report->trace.status = cpkit::TerminalStatus::numerical_failure;
        }
        *out = report.release();
    });
}
// run_likelihood (harness.cpp:488-550): ranks x problems x inits, per-rank
// fraction of problems with at least one converged init. Each rank's instances
// run as one batch (one CTA per instance).
cpkit_status cpkit_run_likelihood(const char* config_json, cpkit_report** out) {
    if (auto st = require(config_json && out, "cpkit_run_likelihood: null argument")) return st;
    return guarded([&] {
        const Spec spec = spec_from_json(Json::parse(config_json));
        auto report = std::make_unique<cpkit_report>();
        report->kind = "likelihood";
        Json cfg = resolved_json(spec);
        cfg["kind"] = "likelihood";
        report->config = cfg;
        const InitDist dist = resolved_init(spec);
        std::vector<BatchJob> jobs;
        for (int rank : spec.ranks) {
            BatchJob job;
            job.dims = spec.dims;
            job.rank = rank;
            job.gn = spec.optimizer == "gn";
            job.als = spec.als;
            job.gncfg = spec.gn;
            for (int p = 0; p < spec.problems; ++p) {  // build_problem_tensor (harness.cpp:422-431)
                if (spec.family == "matmul") {
                    job.tensors.push_back(matmul_data(spec.matmul_n));
                } else {
                    const std::uint64_t ps = cpkit::problem_seed(spec.seed, rank, p);
                    job.tensors.push_back(reconstruct_host(
                        spec.family == "uniform" ? cpkit::random_model_uniform(spec.dims, rank, ps, spec.fa, spec.fb)
                                                 : cpkit::random_model_gaussian(spec.dims, rank, ps)));
                }
                for (int i = 0; i < spec.inits; ++i) {
                    const std::uint64_t is = cpkit::init_seed(spec.seed, rank, p, i);
                    job.x_index.push_back(p);
                    job.inits.push_back(dist.kind == InitKind::uniform
                                            ? cpkit::random_model_uniform(spec.dims, rank, is, dist.a, dist.b)
                                            : cpkit::random_model_gaussian(spec.dims, rank, is));
                }
            }
            jobs.push_back(std::move(job));
        }
        // every rank's batch in flight at once (one stream each), then collect
        std::vector<cudaStream_t> streams(jobs.size());
        std::vector<std::unique_ptr<TinyRun>> runs(jobs.size());
        for (std::size_t k = 0; k < jobs.size(); ++k) {
            CPK_CUDA(cudaStreamCreateWithFlags(&streams[k], cudaStreamNonBlocking));
            jobs[k].gn ? jobs[k].gncfg.validate() : jobs[k].als.validate();
            runs[k] = tiny_launch(jobs[k], false, streams[k]);
        }
        for (std::size_t k = 0; k < jobs.size(); ++k) {
            std::vector<cpkit_instance> res;
            if (runs[k]) {
                CPK_CUDA(cudaStreamSynchronize(streams[k]));
                res = tiny_collect(*runs[k], nullptr);
            } else {
                res = run_batch(jobs[k], nullptr);
            }
            CPK_CUDA(cudaStreamDestroy(streams[k]));
            cpkit_report::LikRank rr;
            rr.rank = jobs[k].rank;
            int with_success = 0;
            for (int p = 0; p < spec.problems; ++p) {
                std::vector<cpkit_instance> inits(res.begin() + p * spec.inits, res.begin() + (p + 1) * spec.inits);
                int converged = 0;
                for (const auto& r : inits)
                    if (r.status == cpkit::TerminalStatus::converged_residual) ++converged;
                if (converged > 0) ++with_success;
                rr.instances.push_back(std::move(inits));
                rr.converged_inits_per_problem.push_back(converged);
            }
            rr.fraction = static_cast<double>(with_success) / static_cast<double>(spec.problems);
            report->likelihood.push_back(std::move(rr));
        }
        *out = report.release();
    });
}

// run_matmul_protocol (harness.cpp:552-653): three arms per init on the n x n
// matrix-multiplication tensor: ALS with decaying lambda, and ALS warm start
// followed by GN (plain / Armijo). Each arm runs as one batch.
cpkit_status cpkit_run_matmul(const char* config_json, cpkit_report** out) {
    if (auto st = require(config_json && out, "cpkit_run_matmul: null argument")) return st;
    return guarded([&] {
        const Json j = Json::parse(config_json);
        // MatmulProtocolSpec (harness.hpp:53-83, harness.cpp:295-376)
        std::uint64_t n = j.value("n", 2ull);
        int rank = j.value("rank", 7), inits = j.value("inits", 100), threads = j.value("threads", 0);
        const std::uint64_t seed = j.value("seed", 0ull);
        InitDist dist = init_from_json(j);
        if (dist.kind == InitKind::family_default) dist.kind = InitKind::gaussian;
        double als_lambda0 = 0.01, als_decay_factor = 2.0, als_residual_tol = 1e-8;
        int als_decay_every = 100, als_max_sweeps = 20000;
        int warm_sweeps = 200;
        double warm_lambda = 0.01;
        double gn_lambda = 1e-3, gn_residual_tol = 1e-8, gn_cg_tol = 1e-3, success_tol = 1e-5;
        int gn_max_iters = 500;
        if (j.contains("als")) {
            const Json& a = j.at("als");
            als_lambda0 = a.value("lambda0", als_lambda0);
            als_decay_factor = a.value("decay_factor", als_decay_factor);
            als_decay_every = a.value("decay_every", als_decay_every);
            als_max_sweeps = a.value("max_sweeps", als_max_sweeps);
            als_residual_tol = a.value("residual_tol", als_residual_tol);
        }
        if (j.contains("warm")) {
            const Json& w = j.at("warm");
            warm_sweeps = w.value("sweeps", warm_sweeps);
            warm_lambda = w.value("lambda", warm_lambda);
        }
        if (j.contains("gn")) {
            const Json& g = j.at("gn");
            gn_lambda = g.value("lambda", gn_lambda);
            gn_max_iters = g.value("max_iters", gn_max_iters);
            gn_residual_tol = g.value("residual_tol", gn_residual_tol);
            gn_cg_tol = g.value("cg_tol", gn_cg_tol);
        }
        success_tol = j.value("success_tol", success_tol);
        if (n < 1) throw cpkit::InvalidArgument("matmul protocol: n must be >= 1");
        if (rank < 1) throw cpkit::InvalidArgument("matmul protocol: rank must be >= 1");
        if (inits < 1) throw cpkit::InvalidArgument("matmul protocol: inits must be >= 1");
        if (als_lambda0 < 0 || warm_lambda < 0 || gn_lambda < 0)
            throw cpkit::InvalidArgument("matmul protocol: negative lambda");
        if (als_decay_every < 1 || als_max_sweeps < 0 || warm_sweeps < 0 || gn_max_iters < 0)
            throw cpkit::InvalidArgument("matmul protocol: bad iteration counts");

        auto report = std::make_unique<cpkit_report>();
        report->kind = "matmul";
        Json cfg = Json::object();  // MatmulProtocolSpec::resolved_json (harness.cpp:349-376)
        cfg["n"] = static_cast<unsigned long long>(n);
        cfg["rank"] = rank;
        cfg["inits"] = inits;
        cfg["seed"] = static_cast<unsigned long long>(seed);
        cfg["threads"] = resolved_threads(threads);
        cfg["init"] = init_to_json(dist);
        Json ja = Json::object();
        ja["lambda0"] = als_lambda0;
        ja["decay_factor"] = als_decay_factor;
        ja["decay_every"] = als_decay_every;
        ja["max_sweeps"] = als_max_sweeps;
        ja["residual_tol"] = als_residual_tol;
        cfg["als"] = ja;
        Json jw = Json::object();
        jw["sweeps"] = warm_sweeps;
        jw["lambda"] = warm_lambda;
        cfg["warm"] = jw;
        Json jg = Json::object();
        jg["lambda"] = gn_lambda;
        jg["max_iters"] = gn_max_iters;
        jg["residual_tol"] = gn_residual_tol;
        jg["cg_tol"] = gn_cg_tol;
        cfg["gn"] = jg;
        cfg["success_tol"] = success_tol;
        cfg["kind"] = "matmul";
        report->config = cfg;
        report->matmul_n = n;
        report->matmul_rank = rank;

        const std::uint64_t sq = n * n;
        const std::vector<std::uint64_t> dims{sq, sq, sq};
        BatchJob base;
        base.dims = dims;
        base.rank = rank;
        base.tensors.push_back(matmul_data(n));
        for (int i = 0; i < inits; ++i) {
            const std::uint64_t is = cpkit::init_seed(seed, rank, 0, i);
            base.x_index.push_back(0);
            base.inits.push_back(dist.kind == InitKind::uniform ? cpkit::random_model_uniform(dims, rank, is, dist.a, dist.b)
                                                                : cpkit::random_model_gaussian(dims, rank, is));
        }
        // arm 0: ALS with decaying lambda
        BatchJob als_arm = base;
        als_arm.als.max_sweeps = als_max_sweeps;
        als_arm.als.residual_tol = als_residual_tol;
        als_arm.als.step_tol = 0.0;
        als_arm.als.lambda0 = als_lambda0;
        als_arm.als.decay_factor = als_decay_factor;
        als_arm.als.decay_every = als_decay_every;
        const std::vector<cpkit_instance> r0 = run_batch(als_arm, nullptr);
        // warm start, then the two GN arms from the warm factors
        BatchJob warm = base;
        warm.als.max_sweeps = warm_sweeps;
        warm.als.residual_tol = 0.0;
        warm.als.step_tol = 0.0;
        warm.als.lambda0 = warm_lambda;
        std::vector<std::vector<double>> warm_f;
        const std::vector<cpkit_instance> rw = run_batch(warm, &warm_f);
        BatchJob gn_plain = base;
        gn_plain.gn = true;
        gn_plain.gncfg.max_iters = gn_max_iters;
        gn_plain.gncfg.residual_tol = gn_residual_tol;
        gn_plain.gncfg.step_tol = 0.0;
        gn_plain.gncfg.cg_tol = gn_cg_tol;
        gn_plain.gncfg.schedule = cpkit::RegSchedule::constant(gn_lambda);
        for (int i = 0; i < inits; ++i)
            gn_plain.inits[i] = model_from_stacked(dims, rank, warm_f[i].data());
        BatchJob gn_armijo = gn_plain;
        gn_armijo.gncfg.armijo = cpkit::ArmijoParams{};
        std::vector<cpkit_instance> r1 = run_batch(gn_plain, nullptr);
        std::vector<cpkit_instance> r2 = run_batch(gn_armijo, nullptr);
        for (int i = 0; i < inits; ++i)
            if (rw[i].status == cpkit::TerminalStatus::numerical_failure) {  // warm start threw
                r1[i] = cpkit_instance{};
                r1[i].status = cpkit::TerminalStatus::numerical_failure;
                r2[i] = r1[i];
            }
        const char* names[3] = {"als_decay", "hybrid_gn", "hybrid_gn_armijo"};
        const std::vector<cpkit_instance>* rs[3] = {&r0, &r1, &r2};
        for (int arm = 0; arm < 3; ++arm) {
            cpkit_report::Arm a;
            a.name = names[arm];
            a.success_tol = arm == 0 ? als_residual_tol : success_tol;
            for (int i = 0; i < inits; ++i) {
                if ((*rs[arm])[i].best_residual < a.success_tol) ++a.converged;
                a.inits.push_back((*rs[arm])[i]);
            }
            report->arms.push_back(std::move(a));
        }
        *out = report.release();
    });
}
// run_bench_matvec (selftest.cpp:275-318): the implicit J^T J matvec timed on
// the device over sizes (warm-up, then the fastest of `reps` single launches,
// CUDA events on the solver stream).
cpkit_status cpkit_run_bench_matvec(const char* config_json, cpkit_report** out) {
    if (auto st = require(out != nullptr, "cpkit_run_bench_matvec: null output")) return st;
    return guarded([&] {
        const Json j = parse_config(config_json);
        const std::uint64_t order = j.value("order", 3ull);
        std::vector<std::uint64_t> sizes{200};
        std::vector<int> ranks{100};
        if (j.contains("s")) {
            sizes.clear();
            for (const auto& v : j.at("s").items()) sizes.push_back(v.as_uint());
        }
        if (j.contains("ranks")) {
            ranks.clear();
            for (const auto& v : j.at("ranks").items()) ranks.push_back(static_cast<int>(v.as_int()));
        }
        const int reps = j.value("reps", 5);
        const std::uint64_t seed = j.value("seed", 0ull);
        if (order < 2 || sizes.empty() || ranks.empty() || reps < 1)
            throw cpkit::InvalidArgument("bench: bad configuration");
        auto report = std::make_unique<cpkit_report>();
        report->kind = "bench";
        Json cfg = Json::object();
        cfg["kind"] = "bench";
        cfg["order"] = static_cast<unsigned long long>(order);
        Json js = Json::array(), jr = Json::array();
        for (auto v : sizes) js.push_back(Json(static_cast<unsigned long long>(v)));
        for (int v : ranks) jr.push_back(Json(v));
        cfg["s"] = js;
        cfg["ranks"] = jr;
        cfg["reps"] = reps;
        cfg["seed"] = static_cast<unsigned long long>(seed);
        report->config = cfg;
        cpkit::Context ctx(current_device());
        for (std::uint64_t s : sizes)
            for (int rank : ranks) {
                const std::vector<std::uint64_t> dims(order, s);
                const cpkit::KruskalModel model = cpkit::random_model_gaussian(dims, rank, cpkit::rng_derive(seed, s));
                const cpkit::KruskalModel w =
                    cpkit::random_model_gaussian(dims, rank, cpkit::rng_derive(cpkit::rng_derive(seed, s), rank));
                cpkit::DeviceProblem p(ctx, dims, rank);
                p.set_factors(model);
                p.build_gamma_set();
                std::vector<double> wh(static_cast<std::size_t>(order * s * rank));
                model_to_stacked(w, wh.data());
                cpkit::DevBuf<double> dw(wh.size()), du(wh.size());
                CPK_CUDA(cudaMemcpy(dw.get(), wh.data(), wh.size() * 8, cudaMemcpyHostToDevice));
                p.jtj_matvec(dw.get(), du.get(), 1e-3, cpkit::RegShape::identity);  // warm-up
                double best = 1e300;
                for (int rep = 0; rep < reps; ++rep) {
                    EventPair ev;
                    CPK_CUDA(cudaEventRecord(ev.a, ctx.stream));
                    p.jtj_matvec(dw.get(), du.get(), 1e-3, cpkit::RegShape::identity);
                    CPK_CUDA(cudaEventRecord(ev.b, ctx.stream));
                    best = std::min(best, ev.ms() * 1e-3);
                }
                cpkit_report::BenchRow row;
                row.order = order;
                row.s = s;
                row.rank = rank;
                row.reps = reps;
                row.seconds_per_matvec = best;
                report->bench.push_back(row);
            }
        *out = report.release();
    });
}
// run_selftest_oracle (selftest.cpp:198-271): the implicit device operators
// against dense routes evaluated on the device (kernels_selftest.cu) on small
// seeded instances: matvec vs explicit J^T J, gradient vs central differences,
// J^T J diagonal blocks vs Gamma(n,n) (x) I, CG vs a dense SPD solve, tree vs
// naive MTTKRP with the contraction budget, fast vs dense residual.
cpkit_status cpkit_run_selftest_oracle(const char* config_json, cpkit_report** out) {
    if (auto st = require(out != nullptr, "cpkit_run_selftest_oracle: null output")) return st;
    return guarded([&] {
        const Json j = parse_config(config_json);
        const std::uint64_t seed = j.value("seed", 0ull);
        const int instances = j.value("instances", 20);
        if (instances < 1) throw cpkit::InvalidArgument("selftest: instances must be >= 1");
        auto report = std::make_unique<cpkit_report>();
        report->kind = "selftest";
        Json cfg = Json::object();
        cfg["kind"] = "selftest";
        cfg["seed"] = static_cast<unsigned long long>(seed);
        cfg["instances"] = instances;
        report->config = cfg;
        using cpkit::rng_derive;
        using cpkit::rng_keyed;
        auto random_dims = [](std::uint64_t sd, std::uint64_t salt, std::size_t order, std::uint64_t lo,
                              std::uint64_t hi) {
            std::vector<std::uint64_t> d(order);
            for (std::size_t m = 0; m < order; ++m) d[m] = lo + rng_keyed(sd, salt, m, 7) % (hi - lo + 1);
            return d;
        };
        auto dense_tensor = [](const std::vector<std::uint64_t>& d, std::uint64_t sd) {
            std::uint64_t total = 1;
            for (auto v : d) total *= v;
            std::vector<double> t(total);
            for (std::uint64_t f = 0; f < total; ++f) t[f] = cpkit::rng_gaussian(sd, 0xDD, f);
            return t;
        };
        auto nrm = [](const std::vector<double>& v) {
            double s = 0.0;
            for (double x : v) s += x * x;
            return std::sqrt(s);
        };
        // stacked (row-major factor blocks) -> vec_stack (column-major per factor, modes in order)
        auto vec_stack = [](const std::vector<double>& st, const std::vector<std::uint64_t>& d, int R) {
            std::vector<double> v(st.size());
            std::size_t off = 0;
            for (auto sn : d) {
                for (std::uint64_t i = 0; i < sn; ++i)
                    for (int r = 0; r < R; ++r) v[off + r * sn + i] = st[off + i * R + r];
                off += sn * R;
            }
            return v;
        };
        struct Acc {
            double max_rel = 0.0;
            int n = 0;
            void add(double r) {
                max_rel = std::max(max_rel, r);
                ++n;
            }
        } matvec, grad, diag, cgc, tree, resid;
        int worst_contractions = 0;
        cpkit::Context ctx(current_device());
        for (int k = 0; k < instances; ++k) {
            const std::uint64_t inst = rng_derive(cpkit::rng_mix64(seed), static_cast<std::uint64_t>(k));
            const std::size_t order = 2 + rng_keyed(inst, 1, 0, 0) % 3;
            const auto dims = random_dims(inst, 2, order, 2, 4);
            const int rank = 1 + static_cast<int>(rng_keyed(inst, 3, 0, 0) % 3);
            const cpkit::KruskalModel model = cpkit::random_model_gaussian(dims, rank, rng_derive(inst, 10));
            const std::vector<double> x = dense_tensor(dims, rng_derive(inst, 11));
            cpkit::DeviceProblem p(ctx, dims, rank);
            p.upload_tensor(x.data());
            p.set_factors(model);
            const std::size_t vars = static_cast<std::size_t>(p.stacked_elems());
            cpkit::DevBuf<double> H(vars * vars), dw(vars), du(vars), dfd(vars), dres(1), db(vars), dy(vars);
            // dense row-major copy for the dense routes (the solver's slab has padded rows)
            cpkit::DevBuf<double> dxd(x.size());
            CPK_CUDA(cudaMemcpyAsync(dxd.get(), x.data(), x.size() * 8, cudaMemcpyHostToDevice, ctx.stream));
            cpkit::launch_explicit_jtj(dims, rank, p.factors_device(), H.get(), ctx.stream);
            std::vector<double> h(vars * vars);
            CPK_CUDA(cudaMemcpyAsync(h.data(), H.get(), h.size() * 8, cudaMemcpyDeviceToHost, ctx.stream));
            // (1) matvec vs explicit J^T J
            const cpkit::KruskalModel w = cpkit::random_model_gaussian(dims, rank, rng_derive(inst, 12));
            std::vector<double> ws(vars), us(vars);
            model_to_stacked(w, ws.data());
            CPK_CUDA(cudaMemcpyAsync(dw.get(), ws.data(), vars * 8, cudaMemcpyHostToDevice, ctx.stream));
            p.build_gamma_set();
            p.jtj_matvec(dw.get(), du.get(), 0.0, cpkit::RegShape::identity);
            CPK_CUDA(cudaMemcpyAsync(us.data(), du.get(), vars * 8, cudaMemcpyDeviceToHost, ctx.stream));
            ctx.sync();
            {
                const std::vector<double> wv = vec_stack(ws, dims, rank), got = vec_stack(us, dims, rank);
                std::vector<double> expd(vars, 0.0), diff(vars);
                for (std::size_t a = 0; a < vars; ++a)
                    for (std::size_t b = 0; b < vars; ++b) expd[a] += h[a * vars + b] * wv[b];
                for (std::size_t a = 0; a < vars; ++a) diff[a] = got[a] - expd[a];
                matvec.add(nrm(diff) / nrm(expd));
            }
            // (2) gradient vs central differences (h = 1e-5)
            for (std::size_t n = 0; n < order; ++n) p.mttkrp_naive(static_cast<int>(n));
            p.gradient();
            cpkit::launch_fd_gradient(dims, rank, p.factors_device(), dxd.get(), 1e-5, dfd.get(), ctx.stream);
            std::vector<double> g(vars), fd(vars);
            CPK_CUDA(cudaMemcpyAsync(g.data(), p.G(), vars * 8, cudaMemcpyDeviceToHost, ctx.stream));
            CPK_CUDA(cudaMemcpyAsync(fd.data(), dfd.get(), vars * 8, cudaMemcpyDeviceToHost, ctx.stream));
            ctx.sync();
            {
                double num = 0.0, den = 0.0;
                for (std::size_t a = 0; a < vars; ++a) {
                    num += (g[a] - fd[a]) * (g[a] - fd[a]);
                    den += g[a] * g[a];
                }
                grad.add(std::sqrt(num / den));
            }
            // (3) diagonal blocks of J^T J vs Gamma(n,n) (x) I
            {
                const std::size_t RR = static_cast<std::size_t>(rank) * rank;
                std::vector<double> grams(order * RR), pairs(order * order * RR);
                p.download_gammas(grams.data(), pairs.data());
                double worst = 0.0;
                std::size_t off = 0;
                for (std::size_t n = 0; n < order; ++n) {
                    const std::size_t sz = dims[n] * rank;
                    double num = 0.0, den = 0.0;
                    for (std::size_t a = 0; a < sz; ++a)
                        for (std::size_t b = 0; b < sz; ++b) {
                            const std::size_t ra = a / dims[n], ia = a % dims[n], rb = b / dims[n], ib = b % dims[n];
                            const double e = ia == ib ? pairs[(n * order + n) * RR + ra * rank + rb] : 0.0;
                            const double d = h[(off + a) * vars + off + b] - e;
                            num += d * d;
                            den += e * e;
                        }
                    worst = std::max(worst, std::sqrt(num) / std::sqrt(den));
                    off += sz;
                }
                diag.add(worst);
            }
            // (4) CG vs dense SPD solve of (J^T J + lambda I) v = -vec(g)
            {
                const double lambda = 1e-3;
                cpkit::GnConfig c;
                c.cg_tol = 1e-10;
                c.cg_max_iters = 100000;
                c.schedule = cpkit::RegSchedule::constant(lambda);
                p.cp_cg(lambda, c);
                std::vector<double> v(vars);
                CPK_CUDA(cudaMemcpyAsync(v.data(), p.V(), vars * 8, cudaMemcpyDeviceToHost, ctx.stream));
                const std::vector<double> gv = vec_stack(g, dims, rank);
                std::vector<double> rhs(vars);
                for (std::size_t a = 0; a < vars; ++a) rhs[a] = -gv[a];
                CPK_CUDA(cudaMemcpyAsync(db.get(), rhs.data(), vars * 8, cudaMemcpyHostToDevice, ctx.stream));
                // Cholesky of the vars x vars system (same device LLT as the ALS solves)
                cpkit::DevBuf<double> dl(cpkit::chol_factor_elems(1, static_cast<int>(vars)));
                cpkit::DevBuf<int> dst(1);
                cpkit::launch_chol_batch(H.get(), 1, static_cast<int>(vars), &lambda, 0, dl.get(), dst.get(),
                                         ctx.stream);
                cpkit::launch_chol_solve_rows(dl.get(), static_cast<int>(vars), db.get(), 1, dy.get(), ctx.stream);
                int stat = 0;
                CPK_CUDA(cudaMemcpyAsync(&stat, dst.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
                std::vector<double> dense(vars);
                CPK_CUDA(cudaMemcpyAsync(dense.data(), dy.get(), vars * 8, cudaMemcpyDeviceToHost, ctx.stream));
                ctx.sync();
                if (stat == 2) throw cpkit::SingularSystem("selftest: dense J^T J + lambda I not positive definite");
                const std::vector<double> vv = vec_stack(v, dims, rank);
                std::vector<double> diff(vars);
                for (std::size_t a = 0; a < vars; ++a) diff[a] = vv[a] - dense[a];
                cgc.add(nrm(diff) / nrm(dense));
            }
            // (6) fast vs dense residual
            {
                const double xn2 = p.norm2();
                p.mttkrp_naive(static_cast<int>(order) - 1);
                p.build_gamma_set();
                const double fast = p.residual_fitness(xn2, static_cast<int>(order) - 1).first;
                cpkit::launch_dense_residual(dims, rank, p.factors_device(), dxd.get(), dres.get(), ctx.stream);
                double dense = 0.0;
                CPK_CUDA(cudaMemcpyAsync(&dense, dres.get(), 8, cudaMemcpyDeviceToHost, ctx.stream));
                ctx.sync();
                resid.add(std::abs(fast - dense));
            }
            // (5) tree vs naive MTTKRP on wider orders, contraction budget
            {
                const std::size_t torder = 3 + rng_keyed(inst, 4, 0, 0) % 3;
                const auto tdims = random_dims(inst, 5, torder, 2, 4);
                const int trank = 2 + static_cast<int>(rng_keyed(inst, 6, 0, 0) % 3);
                const cpkit::KruskalModel tm = cpkit::random_model_gaussian(tdims, trank, rng_derive(inst, 13));
                const std::vector<double> tx = dense_tensor(tdims, rng_derive(inst, 14));
                cpkit::DeviceProblem q(ctx, tdims, trank);
                q.upload_tensor(tx.data());
                cpkit::DevBuf<double> dtx(tx.size());
                CPK_CUDA(cudaMemcpyAsync(dtx.get(), tx.data(), tx.size() * 8, cudaMemcpyHostToDevice, ctx.stream));
                q.set_factors(tm);
                q.invalidate_all();
                q.reset_contraction_counter();
                double worst = 0.0;
                for (std::size_t n = 0; n < torder; ++n) {
                    std::vector<double> a(tdims[n] * trank), b(tdims[n] * trank), d(a.size());
                    q.mttkrp(static_cast<int>(n));
                    q.download_mttkrp(static_cast<int>(n), a.data());
                    cpkit::DevBuf<double> dm(a.size());
                    cpkit::launch_dense_mttkrp(tdims, trank, q.factors_device(), dtx.get(), static_cast<int>(n),
                                               dm.get(), ctx.stream);
                    CPK_CUDA(cudaMemcpyAsync(b.data(), dm.get(), b.size() * 8, cudaMemcpyDeviceToHost, ctx.stream));
                    ctx.sync();
                    for (std::size_t e = 0; e < a.size(); ++e) d[e] = a[e] - b[e];
                    worst = std::max(worst, nrm(d) / nrm(b));
                }
                // budget: a fresh workspace computing every mode
                q.invalidate_all();
                q.reset_contraction_counter();
                for (std::size_t n = 0; n < torder; ++n) q.mttkrp(static_cast<int>(n));
                worst_contractions = std::max(worst_contractions, q.full_contractions());
                tree.add(worst);
            }
        }
        // fault injection for the boundary tests only: scale every tolerance
        // (0 forces the rel-error checks to fail, so cpkit_report_ok must be 0)
        const char* ts = std::getenv("CPKIT_SELFTEST_TOL_SCALE");
        const double tol_scale = ts ? std::atof(ts) : 1.0;
        auto push = [&](const char* name, const Acc& a, double tol) {
            tol *= tol_scale;
            cpkit_report::Check c;
            c.name = name;
            c.instances = a.n;
            c.max_rel_error = a.max_rel;
            c.tolerance = tol;
            c.pass = a.max_rel <= tol;
            report->checks.push_back(c);
        };
        push("hessian_matvec_vs_explicit_jtj", matvec, 1e-12);
        push("gradient_vs_finite_difference", grad, 1e-6);
        push("jtj_diagonal_blocks_vs_kron", diag, 1e-12);
        push("cg_vs_dense_solve", cgc, 1e-6);
        push("tree_mttkrp_vs_naive", tree, 1e-12);
        push("fast_vs_dense_residual", resid, 1e-10);
        cpkit_report::Check budget;
        budget.name = "tree_contraction_budget";
        budget.instances = instances;
        budget.max_rel_error = worst_contractions;
        budget.tolerance = 2.0;
        budget.pass = worst_contractions <= 2;
        report->checks.push_back(budget);
        report->all_pass = true;
        for (const auto& c : report->checks) report->all_pass = report->all_pass && c.pass;
        *out = report.release();
    });
}

// ---- reports ------------------------------------------------------------------------------
cpkit_status cpkit_report_emit(const cpkit_report* r, const char* format, const char* path) {
    if (auto st = require(r && format && path, "cpkit_report_emit: null argument")) return st;
    return guarded([&] {
        std::string payload;
        const std::string f(format);
        if (f == "json") payload = report_to_json(*r).dump(2) + "\n";
        else if (f == "csv") payload = report_to_csv(*r);
        else throw cpkit::InvalidArgument("emit_report: format must be csv or json");
        if (std::string(path) == "-") {
            std::cout << payload;
            std::cout.flush();
            return;
        }
        std::ofstream os(path, std::ios::binary);
        if (!os) throw cpkit::IoError(std::string("cannot open for writing: ") + path);
        os << payload;
        if (!os) throw cpkit::IoError(std::string("write failed: ") + path);
    });
}
cpkit_status cpkit_report_to_json(const cpkit_report* r, char** out_json) {
    if (auto st = require(r && out_json, "cpkit_report_to_json: null argument")) return st;
    return guarded([&] { *out_json = dup_string(report_to_json(*r).dump(2)); });
}
cpkit_status cpkit_report_config(const cpkit_report* r, char** out_json) {
    if (auto st = require(r && out_json, "cpkit_report_config: null argument")) return st;
    return guarded([&] { *out_json = dup_string(r->config.dump(2)); });
}
// cpkit_c.cpp:379-385: a self-test report is OK only when every check passed
int cpkit_report_ok(const cpkit_report* r) {
    if (r == nullptr) return 0;
    if (r->kind == "selftest") return r->all_pass ? 1 : 0;
    return 1;
}
void cpkit_report_destroy(cpkit_report* r) { delete r; }

// ================================================================ device layer
cpkit_status cpkit_dev_problem_create(int device, const uint64_t* dims, uint64_t order, uint64_t rank,
                                      cpkit_dev_problem** out) {
    if (auto st = require(dims && out && order > 0 && rank > 0, "cpkit_dev_problem_create: bad argument")) return st;
    return guarded([&] {
        auto h = std::make_unique<cpkit_dev_problem>();
        h->ctx = std::make_unique<cpkit::Context>(device);
        h->p = std::make_unique<cpkit::DeviceProblem>(*h->ctx, std::vector<std::uint64_t>(dims, dims + order),
                                                      static_cast<int>(rank));
        *out = h.release();
    });
}
cpkit_status cpkit_dev_nccl_unique_id(void* out128) {
    if (auto st = require(out128 != nullptr, "cpkit_dev_nccl_unique_id: null argument")) return st;
    return guarded([&] { cpkit::nccl_unique_id(out128); });
}
cpkit_status cpkit_dev_problem_create_sharded(int device, const uint64_t* dims, uint64_t order, uint64_t rank,
                                              int shard, int world, const void* nccl_id128,
                                              cpkit_dev_problem** out) {
    if (auto st = require(dims && out && order > 0 && rank > 0 && world >= 1 && shard >= 0 && shard < world,
                          "cpkit_dev_problem_create_sharded: bad argument"))
        return st;
    return guarded([&] {
        auto h = std::make_unique<cpkit_dev_problem>();
        h->ctx = std::make_unique<cpkit::Context>(device);
        // world == 1 with an id still routes the collectives through NCCL (a
        // one-rank communicator), which exercises the sharded path on one GPU
        if (world > 1 && !nccl_id128) throw cpkit::InvalidArgument("sharded problem needs an NCCL unique id");
        if (nccl_id128) h->ctx->comm = cpkit::make_nccl_comm(nccl_id128, shard, world);
        h->p = std::make_unique<cpkit::DeviceProblem>(*h->ctx, std::vector<std::uint64_t>(dims, dims + order),
                                                      static_cast<int>(rank));
        *out = h.release();
    });
}
cpkit_status cpkit_dev_problem_create_loopback(int device, const uint64_t* dims, uint64_t order, uint64_t rank,
                                               int world, cpkit_dev_problem** out) {
    if (auto st = require(dims && out && order > 0 && rank > 0 && world >= 1,
                          "cpkit_dev_problem_create_loopback: bad argument"))
        return st;
    return guarded([&] {
        auto comms = cpkit::make_loopback_comms(world);
        std::vector<std::unique_ptr<cpkit_dev_problem>> hs;
        for (int r = 0; r < world; ++r) {
            auto h = std::make_unique<cpkit_dev_problem>();
            h->ctx = std::make_unique<cpkit::Context>(device);
            h->ctx->comm = std::move(comms[r]);
            h->p = std::make_unique<cpkit::DeviceProblem>(*h->ctx, std::vector<std::uint64_t>(dims, dims + order),
                                                          static_cast<int>(rank));
            hs.push_back(std::move(h));
        }
        for (int r = 0; r < world; ++r) out[r] = hs[r].release();
    });
}
void cpkit_dev_problem_destroy(cpkit_dev_problem* p) {
    if (!p) return;
    try {
        p->p.reset();
        p->ctx.reset();
    } catch (...) {
    }
    delete p;
}
cpkit_status cpkit_dev_slab(const cpkit_dev_problem* p, uint64_t* lo, uint64_t* hi, uint64_t* local_elems) {
    if (auto st = require(p && lo && hi && local_elems, "cpkit_dev_slab: null argument")) return st;
    *lo = p->p->slab_lo();
    *hi = p->p->slab_hi();
    *local_elems = p->p->local_elems();
    return CPKIT_OK;
}

#define DEV_REQ(cond) \
    if (auto st_ = require((cond), __func__)) return st_

cpkit_status cpkit_dev_upload_tensor(cpkit_dev_problem* p, const double* host) {
    DEV_REQ(p && host);
    return guarded([&] {
        p->p->upload_tensor(host);
        p->ctx->sync();
    });
}
cpkit_status cpkit_dev_load_tensor(cpkit_dev_problem* p, const char* path) {
    DEV_REQ(p && path);
    return guarded([&] { p->p->load_tensor_file(path); });
}
cpkit_status cpkit_dev_generate_tensor(cpkit_dev_problem* p, const double* truth, uint64_t noise_seed,
                                       double noise_rel) {
    DEV_REQ(p && truth);
    return guarded([&] {
        auto m = model_from_stacked(p->p->dims(), p->p->rank(), truth);
        p->p->generate_tensor(m, noise_seed, noise_rel);
        p->ctx->sync();
    });
}
cpkit_status cpkit_dev_set_factors(cpkit_dev_problem* p, const double* f) {
    DEV_REQ(p && f);
    return guarded([&] {
        p->p->set_factors(model_from_stacked(p->p->dims(), p->p->rank(), f));
        p->ctx->sync();
    });
}
cpkit_status cpkit_dev_get_factors(cpkit_dev_problem* p, double* f) {
    DEV_REQ(p && f);
    return guarded([&] {
        cpkit::KruskalModel m;
        p->p->get_factors(m);
        model_to_stacked(m, f);
    });
}
cpkit_status cpkit_dev_norm2(cpkit_dev_problem* p, double* out) {
    DEV_REQ(p && out);
    return guarded([&] { *out = p->p->norm2(); });
}
cpkit_status cpkit_dev_mttkrp(cpkit_dev_problem* p, uint64_t mode, double* out) {
    DEV_REQ(p);
    return guarded([&] {
        if (mode >= static_cast<uint64_t>(p->p->order())) throw cpkit::InvalidArgument("mttkrp: mode out of range");
        p->p->mttkrp(static_cast<int>(mode));
        if (out) p->p->download_mttkrp(static_cast<int>(mode), out);
        else p->ctx->sync();
    });
}
cpkit_status cpkit_dev_mttkrp_naive(cpkit_dev_problem* p, uint64_t mode, double* out) {
    DEV_REQ(p);
    return guarded([&] {
        if (mode >= static_cast<uint64_t>(p->p->order())) throw cpkit::InvalidArgument("mttkrp: mode out of range");
        p->p->mttkrp_naive(static_cast<int>(mode));
        if (out) p->p->download_mttkrp(static_cast<int>(mode), out);
        else p->ctx->sync();
    });
}
cpkit_status cpkit_dev_note_factor_update(cpkit_dev_problem* p, uint64_t mode) {
    DEV_REQ(p);
    return guarded([&] { p->p->note_factor_update(static_cast<int>(mode)); });
}
int cpkit_dev_full_contractions(const cpkit_dev_problem* p) { return p ? p->p->full_contractions() : 0; }
void cpkit_dev_reset_contraction_counter(cpkit_dev_problem* p) {
    if (p) p->p->reset_contraction_counter();
}
cpkit_status cpkit_dev_gamma_set(cpkit_dev_problem* p, double* grams, double* pair) {
    DEV_REQ(p);
    return guarded([&] {
        p->p->build_gamma_set();
        const int N = p->p->order();
        const std::size_t RR = static_cast<std::size_t>(p->p->rank()) * p->p->rank();
        std::vector<double> g(N * RR), pr(static_cast<std::size_t>(N) * N * RR);
        p->p->download_gammas(g.data(), pr.data());
        if (grams) std::memcpy(grams, g.data(), g.size() * 8);
        if (pair) std::memcpy(pair, pr.data(), pr.size() * 8);
    });
}
cpkit_status cpkit_dev_set_gamma_set(cpkit_dev_problem* p, const double* grams, const double* pair) {
    DEV_REQ(p && grams && pair);
    return guarded([&] {
        p->p->upload_gammas(grams, pair);
        p->ctx->sync();
    });
}
cpkit_status cpkit_dev_residual(cpkit_dev_problem* p, double xnorm2, double* r, double* f) {
    DEV_REQ(p && r && f);
    return guarded([&] {
        p->p->build_gamma_set();
        auto rf = p->p->residual_fitness(xnorm2, p->p->order() - 1);
        *r = rf.first;
        *f = rf.second;
    });
}
namespace {
void upload_stacked(cpkit_dev_problem* p, double* dev, const double* host) {
    CPK_CUDA(cudaMemcpyAsync(dev, host, p->p->stacked_elems() * 8, cudaMemcpyHostToDevice, p->ctx->stream));
}
void download_stacked(cpkit_dev_problem* p, double* host, const double* dev) {
    CPK_CUDA(cudaMemcpyAsync(host, dev, p->p->stacked_elems() * 8, cudaMemcpyDeviceToHost, p->ctx->stream));
    p->ctx->sync();
}
}  // namespace
cpkit_status cpkit_dev_gradient(cpkit_dev_problem* p, const double* mttkrps, double* g_out) {
    DEV_REQ(p && g_out);
    return guarded([&] {
        if (mttkrps) {
            // load caller M into the device M buffer (mode blocks are contiguous)
            CPK_CUDA(cudaMemcpyAsync(const_cast<double*>(p->p->mttkrp_result(0)), mttkrps,
                                     p->p->stacked_elems() * 8, cudaMemcpyHostToDevice, p->ctx->stream));
        }
        p->p->gradient();
        download_stacked(p, g_out, p->p->G());
    });
}
cpkit_status cpkit_dev_jtj_matvec(cpkit_dev_problem* p, const double* w, double lambda, int shape, double* u) {
    DEV_REQ(p && w && u);
    return guarded([&] {
        upload_stacked(p, p->p->Wbuf(), w);
        p->p->jtj_matvec(p->p->Wbuf(), p->p->Ubuf(), lambda,
                         shape == 0 ? cpkit::RegShape::identity : cpkit::RegShape::diagonal);
        download_stacked(p, u, p->p->Ubuf());
    });
}
cpkit_status cpkit_dev_preconditioner(cpkit_dev_problem* p, double lambda, int shape, double* out) {
    DEV_REQ(p && out);
    return guarded([&] {
        p->p->build_preconditioner(lambda, shape == 0 ? cpkit::RegShape::identity : cpkit::RegShape::diagonal);
        const std::size_t n = static_cast<std::size_t>(p->p->order()) * p->p->rank() * p->p->rank();
        CPK_CUDA(cudaMemcpyAsync(out, p->p->pinv(), n * 8, cudaMemcpyDeviceToHost, p->ctx->stream));
        p->ctx->sync();
    });
}
cpkit_status cpkit_dev_cp_cg(cpkit_dev_problem* p, const double* g, double lambda, const char* gn_json,
                             double* v_out, int* iterations, int* hit_cap, int* breakdown) {
    DEV_REQ(p && g && v_out);
    return guarded([&] {
        const cpkit::GnConfig cfg = gn_json ? gn_from_block(Json::parse(gn_json)) : cpkit::GnConfig{};
        cfg.validate();
        upload_stacked(p, p->p->G(), g);
        const cpkit::CgResultInfo r = p->p->cp_cg(lambda, cfg);
        download_stacked(p, v_out, p->p->V());
        if (iterations) *iterations = r.iterations;
        if (hit_cap) *hit_cap = r.hit_cap;
        if (breakdown) *breakdown = r.breakdown;
    });
}
cpkit_status cpkit_dev_spd_solve(cpkit_dev_problem* p, const double* s, const double* b, uint64_t rows,
                                 double lambda, double* y) {
    DEV_REQ(p && s && b && y);
    return guarded([&] {
        const int R = p->p->rank();
        const std::size_t rr = static_cast<std::size_t>(R) * R;
        cpkit::DevBuf<double> ds(rr), db(rows * R), dy(rows * R);
        CPK_CUDA(cudaMemcpyAsync(ds.get(), s, rr * 8, cudaMemcpyHostToDevice, p->ctx->stream));
        CPK_CUDA(cudaMemcpyAsync(db.get(), b, rows * R * 8, cudaMemcpyHostToDevice, p->ctx->stream));
        p->p->spd_solve(ds.get(), db.get(), static_cast<std::int64_t>(rows), lambda, dy.get());
        CPK_CUDA(cudaMemcpyAsync(y, dy.get(), rows * R * 8, cudaMemcpyDeviceToHost, p->ctx->stream));
        p->ctx->sync();
    });
}
cpkit_status cpkit_dev_spd_inverse(cpkit_dev_problem* p, const double* s, double lambda, double* inv) {
    DEV_REQ(p && s && inv);
    return guarded([&] {
        const int R = p->p->rank();
        const std::size_t rr = static_cast<std::size_t>(R) * R;
        cpkit::DevBuf<double> ds(rr), di(rr);
        CPK_CUDA(cudaMemcpyAsync(ds.get(), s, rr * 8, cudaMemcpyHostToDevice, p->ctx->stream));
        p->p->spd_inverse(ds.get(), lambda, di.get());
        CPK_CUDA(cudaMemcpyAsync(inv, di.get(), rr * 8, cudaMemcpyDeviceToHost, p->ctx->stream));
        p->ctx->sync();
    });
}
cpkit_status cpkit_dev_als_sweep(cpkit_dev_problem* p, double lambda, double* step_norm, int* contractions) {
    DEV_REQ(p);
    return guarded([&] {
        const cpkit::AlsSweepDiag d = p->p->als_sweep(lambda);
        if (step_norm) *step_norm = d.step_norm;
        if (contractions) *contractions = d.full_contractions;
    });
}
cpkit_status cpkit_dev_gn_step(cpkit_dev_problem* p, const char* gn_json, double xnorm2, double* diag12) {
    DEV_REQ(p && diag12);
    return guarded([&] {
        const cpkit::GnConfig cfg = gn_json ? gn_from_block(Json::parse(gn_json)) : cpkit::GnConfig{};
        cfg.validate();
        cpkit::RegSchedule s = cfg.schedule;
        const cpkit::GnStepDiag d = p->p->gn_step(cfg, s, xnorm2);
        const double v[12] = {static_cast<double>(d.halt), double(d.stepped), d.residual_before, d.residual_after,
                              d.grad_norm, d.lambda, double(d.cg_iters), d.step_norm, d.alpha,
                              double(d.armijo_exhausted), double(d.cg_hit_cap), double(d.cg_breakdown)};
        std::memcpy(diag12, v, sizeof v);
    });
}
cpkit_status cpkit_dev_optimize(cpkit_dev_problem* p, const char* config_json, const double* init,
                                double* out_factors, cpkit_report** out_report) {
    DEV_REQ(p);
    return guarded([&] {
        const Json j = parse_config(config_json);
        const std::string optimizer = j.value("optimizer", "als");
        Json wrapped = j;
        Json prob = Json::object();
        prob["family"] = "gaussian";
        Json dims = Json::array();
        for (auto d : p->p->dims()) dims.push_back(Json(static_cast<unsigned long long>(d)));
        prob["dims"] = dims;
        prob["rank"] = p->p->rank();
        wrapped["problem"] = prob;
        const Spec spec = spec_from_json(wrapped);
        cpkit::KruskalModel start;
        if (init) {
            start = model_from_stacked(p->p->dims(), p->p->rank(), init);
        } else {
            Json jr = j;
            jr["rank"] = p->p->rank();
            start = start_model(p->p->dims(), jr, spec);
        }
        auto report = std::make_unique<cpkit_report>();
        Json cfg = resolved_json(spec);
        cfg["kind"] = "decompose";
        cfg["optimizer"] = optimizer;
        report->config = cfg;
        cpkit::KruskalModel result;
        run_optimizer(*p->p, optimizer, spec, std::move(start), result, *report);
        if (out_factors) model_to_stacked(result, out_factors);
        if (out_report) *out_report = report.release();
    });
}

// ---- timing ----------------------------------------------------------------------------
cpkit_status cpkit_dev_time_als_sweeps(cpkit_dev_problem* p, double lambda, int sweeps, double* ms) {
    DEV_REQ(p && ms && sweeps > 0);
    return guarded([&] {
        EventPair ev;
        // each sweep's diagnostics are read back (as the driver does), with
        // the next sweep already queued behind it
        CPK_CUDA(cudaEventRecord(ev.a, p->ctx->stream));
        for (int i = 0; i < sweeps; ++i) {
            p->p->als_sweep_launch(lambda, false);
            if (p->p->als_sweeps_pending() > 1) p->p->als_sweep_finish();
        }
        while (p->p->als_sweeps_pending() > 0) p->p->als_sweep_finish();
        CPK_CUDA(cudaEventRecord(ev.b, p->ctx->stream));
        *ms = ev.ms();
    });
}
cpkit_status cpkit_dev_time_roots(cpkit_dev_problem* p, int reps, double* ms_back, double* ms_front) {
    DEV_REQ(p && ms_back && ms_front && reps > 0);
    return guarded([&] {
        const int N = p->p->order();
        const int h = (N + 1) / 2;
        p->p->profile_enable(true);
        for (int i = 0; i < reps; ++i) {
            p->p->mttkrp_naive(0);  // back root (+ level 2, not timed)
            p->p->mttkrp_naive(h);  // front root (+ level 2, not timed)
        }
        double ms[3];
        int cnt[3];
        p->p->profile_read(ms, cnt);
        p->p->profile_enable(false);
        *ms_back = cnt[0] ? ms[0] / cnt[0] : 0.0;
        *ms_front = cnt[1] ? ms[1] / cnt[1] : 0.0;
    });
}
cpkit_status cpkit_dev_profile(cpkit_dev_problem* p, int enable) {
    DEV_REQ(p);
    return guarded([&] { p->p->profile_enable(enable != 0); });
}
cpkit_status cpkit_dev_profile_read(cpkit_dev_problem* p, double* ms3, int* count3) {
    DEV_REQ(p && ms3 && count3);
    return guarded([&] { p->p->profile_read(ms3, count3); });
}
cpkit_status cpkit_dev_time_jtj(cpkit_dev_problem* p, int reps, double* ms) {
    DEV_REQ(p && ms && reps > 0);
    return guarded([&] {
        p->p->build_gamma_set();
        EventPair ev;
        CPK_CUDA(cudaEventRecord(ev.a, p->ctx->stream));
        for (int i = 0; i < reps; ++i)
            p->p->jtj_matvec(p->p->factors_device(), p->p->Ubuf(), 1e-3, cpkit::RegShape::identity);
        CPK_CUDA(cudaEventRecord(ev.b, p->ctx->stream));
        *ms = ev.ms() / reps;
    });
}
cpkit_status cpkit_dev_time_norm2(cpkit_dev_problem* p, int reps, double* ms) {
    DEV_REQ(p && ms && reps > 0);
    return guarded([&] {
        EventPair ev;
        CPK_CUDA(cudaEventRecord(ev.a, p->ctx->stream));
        for (int i = 0; i < reps; ++i) p->p->norm2();
        CPK_CUDA(cudaEventRecord(ev.b, p->ctx->stream));
        *ms = ev.ms() / reps;
    });
}
cpkit_status cpkit_dev_time_second_level(cpkit_dev_problem* p, int reps, double* ms, double* bytes) {
    DEV_REQ(p && ms && bytes && reps > 0);
    return guarded([&] { *ms = p->p->time_second_level(reps, bytes); });
}
cpkit_status cpkit_dev_probe_dmma_peak(int device, double* tflops) {
    DEV_REQ(tflops);
    return guarded([&] { *tflops = cpkit::probe_dmma_peak(device); });
}
uint64_t cpkit_dev_kernel_launches(void) { return cpkit::kernel_launches(); }
uint64_t cpkit_dev_guard_violations(void) { return cpkit::guard_violations(); }
cpkit_status cpkit_dev_guard_selftest(int* detected) {
    if (!detected) return fail(CPKIT_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] { *detected = cpkit::guard_selftest() ? 1 : 0; });
}

cpkit_status cpkit_dev_random_factors(const uint64_t* dims, uint64_t order, uint64_t rank, uint64_t seed,
                                      int kind, double a, double b, double* out) {
    DEV_REQ(dims && out && order > 0 && rank > 0);
    return guarded([&] {
        std::vector<std::uint64_t> d(dims, dims + order);
        const auto m = kind == 0 ? cpkit::random_model_uniform(d, static_cast<std::int64_t>(rank), seed, a, b)
                                 : cpkit::random_model_gaussian(d, static_cast<std::int64_t>(rank), seed);
        model_to_stacked(m, out);
    });
}
cpkit_status cpkit_dev_shard_range(uint64_t extent, int shard, int world, uint64_t* lo, uint64_t* hi) {
    DEV_REQ(lo && hi && world >= 1 && shard >= 0 && shard < world);
    cpkit::shard_range(extent, shard, world, lo, hi);
    return CPKIT_OK;
}
uint64_t cpkit_dev_problem_seed(uint64_t master, int rank, int problem) {
    return cpkit::problem_seed(master, rank, problem);
}
uint64_t cpkit_dev_init_seed(uint64_t master, int rank, int problem, int init) {
    return cpkit::init_seed(master, rank, problem, init);
}
cpkit_status cpkit_dev_download_tensor(cpkit_dev_problem* p, double* host_local) {
    DEV_REQ(p && host_local);
    return guarded([&] {
        p->p->download_tensor(host_local);
    });
}
cpkit_status cpkit_dev_time_gn_steps(cpkit_dev_problem* p, const char* gn_json, int steps, double* ms,
                                     int* cg_iters_total) {
    DEV_REQ(p && ms && steps > 0);
    return guarded([&] {
        const cpkit::GnConfig cfg = gn_json ? gn_from_block(Json::parse(gn_json)) : cpkit::GnConfig{};
        cfg.validate();
        cpkit::RegSchedule s = cfg.schedule;
        const double xn2 = p->p->norm2();
        p->p->prepare_gn();  // the starting point's tree pass (gn_optimize's setup), untimed
        int cg = 0;
        EventPair ev;
        CPK_CUDA(cudaEventRecord(ev.a, p->ctx->stream));
        if (!cfg.armijo && !std::getenv("CPKIT_GN_SYNC") && !std::getenv("CPKIT_GN_NO_PIPELINE")) {
            // gn_optimize's pipelined loop: step k+1 queued before step k is read
            int slot = 0;
            p->p->gn_enqueue(cfg, s, xn2, slot);
            for (int i = 0; i < steps; ++i) {
                const cpkit::RegSchedule next = cpkit::schedule_next(s);
                const bool spec = i + 1 < steps;
                if (spec) p->p->gn_enqueue(cfg, next, xn2, slot ^ 1);
                const cpkit::GnStepDiag d = p->p->gn_decode(cfg, s.lambda, slot);
                cg += d.cg_iters;
                if (!d.stepped) {
                    if (spec) p->p->ctx().sync();
                    break;
                }
                s = next;
                slot ^= 1;
            }
        } else {
            for (int i = 0; i < steps; ++i) {
                cpkit::GnStepDiag d = p->p->gn_step(cfg, s, xn2);
                cg += d.cg_iters;
                if (!d.stepped) break;
            }
        }
        CPK_CUDA(cudaEventRecord(ev.b, p->ctx->stream));
        *ms = ev.ms();
        if (cg_iters_total) *cg_iters_total = cg;
    });
}

}  // extern "C"
