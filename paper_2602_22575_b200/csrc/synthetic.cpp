// synthetic.cpp -- host generator of the benchmark's stripe-structured inputs.
//
// Restates generate_synthetic (proj/src/synthetic.cpp:276-328) so the benchmark's
// inputs are the reference's inputs bit for bit (checked by tests/test_synthetic.py
// against the compiled reference), but multi-threaded for 128K x 32-head tensors:
//   * per-(z,h) gaussian background streams run in parallel (as in the reference);
//   * vertical / horizontal planting: geometry drawn once from the shared plant
//     stream, then applied per (z,h) slice in parallel;
//   * slash planting: per-(stripe, position) directions are independent streams, and
//     within one stripe every Q row / K row receives at most one update, so positions
//     are split across threads while stripes stay in order.
// Compiled with -ffp-contract=off so every float/double expression rounds like the
// reference build.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "s2o_cuda.h"

namespace s2o_synth {
namespace {

uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// mix_seed synthetic.cpp:29-36
uint64_t mix_seed(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
    uint64_t x = seed;
    (void)splitmix64(x);
    x ^= splitmix64(x) + a;
    x ^= splitmix64(x) + b;
    x ^= splitmix64(x) + c;
    return splitmix64(x);
}

// xoshiro256** + Box-Muller, synthetic.cpp:38-108
class Rng {
public:
    explicit Rng(uint64_t seed) {
        uint64_t x = seed;
        for (auto& s : s_) s = splitmix64(x);
    }
    uint64_t next_bits() {
        const uint64_t result = rotl(s_[1] * 5, 7) * 9;
        const uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return result;
    }
    double uniform() { return static_cast<double>(next_bits() >> 11) * 0x1.0p-53; }
    double normal() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        const double u1 = static_cast<double>((next_bits() >> 11) + 1) * 0x1.0p-53;
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * std::numbers::pi * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }
    int64_t uniform_int(int64_t n) {
        if (n <= 0) throw std::invalid_argument("uniform_int needs n > 0");
        return static_cast<int64_t>(next_bits() % static_cast<uint64_t>(n));
    }
    std::vector<int64_t> sample_distinct(int64_t count, int64_t n) {
        if (count > n) throw std::invalid_argument("cannot sample more distinct values than the domain holds");
        std::unordered_set<int64_t> seen;
        std::vector<int64_t> out;
        out.reserve(static_cast<size_t>(count));
        while (static_cast<int64_t>(out.size()) < count) {
            const int64_t v = uniform_int(n);
            if (seen.insert(v).second) out.push_back(v);
        }
        return out;
    }
    std::vector<double> unit_direction(int64_t d) {
        std::vector<double> dir(static_cast<size_t>(d));
        double norm_sq = 0.0;
        for (auto& x : dir) {
            x = normal();
            norm_sq += x * x;
        }
        const double inv = 1.0 / std::sqrt(norm_sq);
        for (auto& x : dir) x *= inv;
        return dir;
    }

private:
    uint64_t s_[4];
    bool have_spare_ = false;
    double spare_ = 0.0;
};

constexpr uint64_t kBaseStream = 0x5b17;
constexpr uint64_t kPlantStream = 0x9a42;
constexpr uint64_t kSlashStream = 0xd3f1;

struct View {
    float* q;
    float* k;
    float* v;
    int64_t z, h, l, d;
    float* row(float* t, int64_t slice, int64_t i) const { return t + (slice * l + i) * d; }
};

template <typename F>
void parallel_for(int64_t count, int threads, F&& fn) {
    const int64_t workers = std::max<int64_t>(1, std::min<int64_t>(threads, count));
    if (workers <= 1) {
        for (int64_t i = 0; i < count; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int64_t w = 0; w < workers; ++w) {
        const int64_t lo = count * w / workers, hi = count * (w + 1) / workers;
        pool.emplace_back([&, lo, hi] {
            for (int64_t i = lo; i < hi; ++i) fn(i);
        });
    }
    for (auto& t : pool) t.join();
}

void add_scaled(float* row, const std::vector<double>& dir, double scale) {
    for (size_t i = 0; i < dir.size(); ++i)
        row[i] = static_cast<float>(static_cast<double>(row[i]) + scale * dir[i]);
}

void set_component(float* row, const std::vector<double>& dir, double target, int64_t d) {
    double current = 0.0;
    for (int64_t i = 0; i < d; ++i) current += static_cast<double>(row[i]) * dir[static_cast<size_t>(i)];
    add_scaled(row, dir, target - current);
}

double stripe_amp(double gain, int64_t d) { return std::sqrt(gain * std::sqrt(static_cast<double>(d))); }

// plant_vertical synthetic.cpp:165-196 / plant_horizontal synthetic.cpp:202-243
void plant_rows(const View& t, const std::vector<double>& dir, double amp,
                const std::vector<double>* row_scale, const std::vector<int64_t>& keys,
                const std::vector<double>& key_scale, int threads) {
    std::vector<uint8_t> planted(static_cast<size_t>(t.l), 0);
    for (int64_t j : keys) planted[static_cast<size_t>(j)] = 1;
    if (!(amp > 0.0)) return;
    parallel_for(t.z * t.h, threads, [&](int64_t slice) {
        for (int64_t i = 0; i < t.l; ++i) {
            const double target = row_scale ? amp * (*row_scale)[static_cast<size_t>(i)] : amp;
            set_component(t.row(t.q, slice, i), dir, target, t.d);
        }
        for (int64_t j = 0; j < t.l; ++j)
            if (!planted[static_cast<size_t>(j)]) set_component(t.row(t.k, slice, j), dir, 0.0, t.d);
        for (size_t s = 0; s < keys.size(); ++s)
            set_component(t.row(t.k, slice, keys[s]), dir, amp * key_scale[s], t.d);
    });
}

void plant_vertical(const View& t, int64_t stripes, double gain, Rng& plant, int threads) {
    const double amp = stripe_amp(gain, t.d);
    const std::vector<int64_t> keys = plant.sample_distinct(stripes, t.l);
    const std::vector<double> dir = plant.unit_direction(t.d);
    std::vector<double> key_scale(keys.size());
    for (double& s : key_scale) s = 0.5 + 0.5 * plant.uniform();
    plant_rows(t, dir, amp, nullptr, keys, key_scale, threads);
}

void plant_horizontal(const View& t, int64_t stripes, double gain, Rng& plant, int threads) {
    const double amp = stripe_amp(gain, t.d);
    const std::vector<int64_t> keys = plant.sample_distinct(stripes, t.l);
    const std::vector<int64_t> rows = plant.sample_distinct(stripes, t.l);
    const std::vector<double> dir = plant.unit_direction(t.d);
    std::vector<double> key_scale(keys.size());
    for (double& s : key_scale) s = 0.5 + 0.5 * plant.uniform();
    std::vector<double> row_scale(static_cast<size_t>(t.l));
    for (double& s : row_scale) s = 0.55 + 0.35 * plant.uniform();
    for (int64_t i : rows) row_scale[static_cast<size_t>(i)] = 1.0;
    plant_rows(t, dir, amp, &row_scale, keys, key_scale, threads);
}

// plant_slash synthetic.cpp:247-272
void plant_slash(const View& t, int64_t stripes, double gain, uint64_t seed, Rng& plant,
                 int threads) {
    const int64_t max_offset = std::max<int64_t>(1, t.l / 8);
    std::vector<int64_t> offsets;
    std::vector<double> stripe_scale;
    for (int64_t s = 0; s < stripes; ++s) {
        offsets.push_back(1 + plant.uniform_int(max_offset));
        stripe_scale.push_back(0.6 + 0.4 * plant.uniform());
    }
    for (size_t s = 0; s < offsets.size() && gain > 0.0; ++s) {
        const int64_t delta = offsets[s];
        const double amp = stripe_amp(gain * stripe_scale[s], t.d);
        const int64_t count = t.l - delta;
        if (count <= 0) continue;
        const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(count, int64_t(threads) * 8));
        parallel_for(chunks, threads, [&](int64_t c) {
            const int64_t lo = delta + count * c / chunks, hi = delta + count * (c + 1) / chunks;
            for (int64_t i = lo; i < hi; ++i) {
                Rng dir_rng(mix_seed(seed, kSlashStream, static_cast<uint64_t>(s), static_cast<uint64_t>(i)));
                const std::vector<double> dir = dir_rng.unit_direction(t.d);
                for (int64_t slice = 0; slice < t.z * t.h; ++slice) {
                    add_scaled(t.row(t.q, slice, i), dir, amp);
                    add_scaled(t.row(t.k, slice, i - delta), dir, amp);
                }
            }
        });
    }
}

}  // namespace
}  // namespace s2o_synth

extern "C" s2o_status s2o_synthetic_generate(const char* pattern, int64_t stripe_count,
                                             double stripe_gain, uint64_t seed, int64_t z,
                                             int64_t h, int64_t l, int64_t d, float* q, float* k,
                                             float* v, int32_t threads) {
    using namespace s2o_synth;
    if (!pattern || !q || !k || !v || z < 1 || h < 1 || l < 1 || d < 1) return S2O_ERR_INVALID_ARG;
    const std::string p(pattern);
    int kind;
    if (p == "gaussian") kind = 0;
    else if (p == "vertical" || p == "vertical-stripes") kind = 1;
    else if (p == "horizontal" || p == "horizontal-stripes") kind = 2;
    else if (p == "slash" || p == "slash-stripes") kind = 3;
    else if (p == "mixed") kind = 4;
    else return S2O_ERR_INVALID_ARG;  // "unknown pattern"
    if (kind != 0 && stripe_count >= l) return S2O_ERR_INVALID_ARG;  // "dims too small for stripe_count"
    if (!std::isfinite(stripe_gain)) return S2O_ERR_INVALID_ARG;
    int nt = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    View t{q, k, v, z, h, l, d};
    parallel_for(z * h, nt, [&](int64_t slice) {
        const int64_t zi = slice / h, hi = slice % h;
        Rng rng(mix_seed(seed, kBaseStream, static_cast<uint64_t>(zi), static_cast<uint64_t>(hi)));
        for (float* base : {q, k, v}) {
            float* row = base + slice * l * d;
            for (int64_t i = 0; i < l * d; ++i) row[i] = static_cast<float>(rng.normal());
        }
    });
    Rng plant(mix_seed(seed, kPlantStream));
    try {
        switch (kind) {
            case 1: plant_vertical(t, stripe_count, stripe_gain, plant, nt); break;
            case 2: plant_horizontal(t, stripe_count, stripe_gain, plant, nt); break;
            case 3: plant_slash(t, stripe_count, stripe_gain, seed, plant, nt); break;
            case 4:
                plant_vertical(t, stripe_count, stripe_gain, plant, nt);
                plant_horizontal(t, stripe_count, stripe_gain, plant, nt);
                plant_slash(t, std::min<int64_t>(2, stripe_count), 0.5 * stripe_gain, seed, plant, nt);
                break;
            default: break;
        }
    } catch (const std::exception&) {
        return S2O_ERR_INVALID_ARG;
    }
    return S2O_OK;
}
