// Calibration of the co-run penalties from measured C3 speedups — how the B200
// runtime's predictor is fitted to what bench/sweep runs measure.
//
// Contract follows the reference (/root/reference/proj/src/calibrate.cpp:34-238):
// measured CSV "scenario_id,collective,strategy,measured_speedup"; FitError for
// fewer than 3 samples or fewer than 2 concurrent strategies; UnknownEntityError
// for a sample naming an unknown scenario; penalties stay feasible (>= 1 and
// DMA <= CU per class). The solver here is a damped Gauss-Newton
// (Levenberg-Marquardt) on the 8 penalties with a forward-difference Jacobian
// and a Cholesky solve of the damped normal equations.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

#include "c3sim/calibrate.hpp"
#include "c3sim/errors.hpp"

namespace c3sim {

namespace {

std::string trimmed(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return {};
    return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}

constexpr int kP = 2 * kNumKernelClasses;
using Vec = std::array<double, kP>;

Vec flatten(const CoRunPenalty& p) {
    Vec v{};
    for (int c = 0; c < kNumKernelClasses; ++c)
        for (int b = 0; b < 2; ++b) v[static_cast<std::size_t>(2 * c + b)] = p.factor[static_cast<std::size_t>(c)][static_cast<std::size_t>(b)];
    return v;
}

CoRunPenalty unflatten(const Vec& v) {
    CoRunPenalty p;
    for (int c = 0; c < kNumKernelClasses; ++c)
        for (int b = 0; b < 2; ++b) p.factor[static_cast<std::size_t>(c)][static_cast<std::size_t>(b)] = v[static_cast<std::size_t>(2 * c + b)];
    return p;
}

bool feasible(const Vec& v) {
    for (int c = 0; c < kNumKernelClasses; ++c) {
        const double cu = v[static_cast<std::size_t>(2 * c)], dma = v[static_cast<std::size_t>(2 * c + 1)];
        if (cu < 1.0 || dma < 1.0 || dma > cu) return false;
    }
    return true;
}

// Solve (A) x = b for symmetric positive definite A; false when not SPD.
bool cholesky_solve(std::array<Vec, kP> A, Vec b, Vec& x) {
    for (int j = 0; j < kP; ++j) {
        double d = A[j][j];
        for (int k = 0; k < j; ++k) d -= A[j][k] * A[j][k];
        if (!(d > 1e-300)) return false;
        A[j][j] = std::sqrt(d);
        for (int i = j + 1; i < kP; ++i) {
            double s = A[i][j];
            for (int k = 0; k < j; ++k) s -= A[i][k] * A[j][k];
            A[i][j] = s / A[j][j];
        }
    }
    for (int i = 0; i < kP; ++i) {  // L y = b
        for (int k = 0; k < i; ++k) b[i] -= A[i][k] * b[k];
        b[i] /= A[i][i];
    }
    for (int i = kP - 1; i >= 0; --i) {  // L^T x = y
        for (int k = i + 1; k < kP; ++k) b[i] -= A[k][i] * b[k];
        b[i] /= A[i][i];
    }
    x = b;
    return true;
}

}  // namespace

std::vector<MeasuredSample> parse_measured_csv(const std::string& text) {
    std::istringstream in(text);
    std::string line;
    if (!std::getline(in, line) || trimmed(line) != "scenario_id,collective,strategy,measured_speedup")
        throw ValidationError(
            "measured csv: expected header scenario_id,collective,strategy,measured_speedup");
    std::vector<MeasuredSample> out;
    for (int lineno = 2; std::getline(in, line); ++lineno) {
        const std::string row = trimmed(line);
        if (row.empty()) continue;
        std::vector<std::string> cells;
        std::istringstream cs(row);
        for (std::string c; std::getline(cs, c, ',');) cells.push_back(c);
        const std::string at = " at line " + std::to_string(lineno);
        if (cells.size() < 4) throw ValidationError("measured csv: malformed row" + at);
        if (cells.size() > 4) throw ValidationError("measured csv: too many cells" + at);
        MeasuredSample s;
        s.scenario_id = trimmed(cells[0]);
        s.collective = collective_kind_from_string(trimmed(cells[1]));
        s.strategy = strategy_from_string(trimmed(cells[2]));
        try {
            s.measured_speedup = std::stod(trimmed(cells[3]));
        } catch (const std::exception&) {
            throw ValidationError("measured csv: bad speedup" + at);
        }
        if (!(s.measured_speedup > 0)) throw ValidationError("measured csv: speedup must be > 0" + at);
        out.push_back(std::move(s));
    }
    return out;
}

std::vector<MeasuredSample> load_measured_csv(const std::filesystem::path& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open file: " + path.string());
    std::ostringstream os;
    os << f.rdbuf();
    return parse_measured_csv(os.str());
}

FitResult fit_penalties(const std::vector<C3Scenario>& scenarios,
                        const std::vector<MeasuredSample>& samples,
                        const MachineDescriptor& md, const SlowdownTableSet& tables,
                        const EfficiencyParams& params, const CoRunPenalty& initial) {
    if (samples.size() < 3)
        throw FitError("calibration needs at least 3 measured samples, got " +
                       std::to_string(samples.size()));
    std::set<Strategy> concurrent;
    for (const auto& s : samples)
        if (s.strategy != Strategy::Serial) concurrent.insert(s.strategy);
    if (concurrent.size() < 2)
        throw FitError("calibration needs samples from at least 2 concurrent strategies");
    std::map<std::pair<std::string, CollectiveKind>, const C3Scenario*> by_key;
    for (const auto& s : scenarios) by_key[{s.id, s.collective.kind}] = &s;
    std::vector<const C3Scenario*> target;
    for (const auto& s : samples) {
        const auto it = by_key.find({s.scenario_id, s.collective});
        if (it == by_key.end())
            throw UnknownEntityError("measured csv references unknown scenario '" + s.scenario_id +
                                     "' (" + to_string(s.collective) + ")");
        target.push_back(it->second);
    }
    const std::size_t m = samples.size();
    const auto resid = [&](const Vec& v, std::vector<double>& r) {
        if (!feasible(v)) {  // keep the search inside the feasible set
            std::fill(r.begin(), r.end(), 1e6);
            return;
        }
        const CoRunPenalty p = unflatten(v);
        for (std::size_t i = 0; i < m; ++i)
            r[i] = simulate(*target[i], samples[i].strategy, md, tables, p, params).speedup -
                   samples[i].measured_speedup;
    };
    const auto ss = [](const std::vector<double>& r) {
        double s = 0;
        for (double v : r) s += v * v;
        return s;
    };

    Vec theta = flatten(initial);
    std::vector<double> r(m), rt(m);
    resid(theta, r);
    double cost = ss(r), damping = 1e-3;
    int it = 0;
    for (; it < 200; ++it) {
        std::vector<Vec> J(m);
        for (int j = 0; j < kP; ++j) {
            Vec t = theta;
            double h = 1e-6;
            t[j] += h;
            if (!feasible(t)) {
                h = -h;
                t[j] = theta[j] + h;
            }
            if (!feasible(t)) {
                for (auto& row : J) row[j] = 0.0;
                continue;
            }
            resid(t, rt);
            for (std::size_t i = 0; i < m; ++i) J[i][j] = (rt[i] - r[i]) / h;
        }
        std::array<Vec, kP> JtJ{};
        Vec Jtr{};
        for (std::size_t i = 0; i < m; ++i)
            for (int a = 0; a < kP; ++a) {
                Jtr[a] += J[i][a] * r[i];
                for (int b = 0; b < kP; ++b) JtJ[a][b] += J[i][a] * J[i][b];
            }
        bool stepped = false;
        for (int attempt = 0; attempt < 8 && !stepped; ++attempt) {
            auto A = JtJ;
            for (int a = 0; a < kP; ++a) A[a][a] += damping * (JtJ[a][a] + 1e-12);
            Vec neg{}, dx{};
            for (int a = 0; a < kP; ++a) neg[a] = -Jtr[a];
            const bool ok = cholesky_solve(A, neg, dx);
            Vec trial = theta;
            for (int a = 0; a < kP; ++a) trial[a] = std::max(1.0, theta[a] + (ok ? dx[a] : 0.0));
            resid(trial, rt);
            const double c2 = ss(rt);
            if (ok && c2 < cost) {
                theta = trial;
                r = rt;
                cost = c2;
                damping = std::max(damping * 0.3, 1e-12);
                stepped = true;
            } else {
                damping *= 10.0;
            }
        }
        if (!stepped || cost < 1e-24) break;
    }
    FitResult fr;
    fr.penalties = unflatten(theta);
    validate(fr.penalties);
    fr.rms_residual = std::sqrt(cost / static_cast<double>(m));
    fr.iterations = it + 1;
    return fr;
}

}  // namespace c3sim
