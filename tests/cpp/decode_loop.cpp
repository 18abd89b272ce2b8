// A C++ host driving the SWA decode through the device-resident mirror
// (include/skv/b200.hpp), no Python anywhere: the way a reference caller
// (Engine::decode_step, engine.hpp:571-684) would run it on a B200.
//
//   decode_loop [layers batch heads prompt steps]
//
// Prompt K/V and the per-step q/k/v live in pinned host buffers (the
// skv_host_alloc helper); every step goes through decode_step_host, so the
// PCIe traffic is inside the timed loop. The same steps also run through the
// device-buffer decode_step on a twin cache and the two must agree bit for
// bit -- outputs and importance -- which checks the host pipeline from C++.
// A third cache runs the steps the way a CPU-side Engine::decode_step would
// feed a GPU attention layer by layer: per layer, synchronous uploads of its
// q / k / v, decode_layer, a synchronous download of its output before the
// next layer (e2e_layer_sync_tokens_per_s; must agree bit for bit too).
// Prints one JSON line; exit 0 = agreement.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "skv/b200.hpp"

namespace {

struct Pinned {
    void* p = nullptr;
    explicit Pinned(std::size_t bytes) { skv::b200::check(skv_host_alloc(bytes, &p)); }
    ~Pinned() { skv_host_free(p); }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// fp32 -> IEEE fp16 bits, round to nearest even (inputs are N(0,1): normal range)
std::uint16_t to_half(float f) {
    std::uint32_t x;
    std::memcpy(&x, &f, 4);
    const std::uint32_t sign = (x >> 16) & 0x8000u;
    const int exp = static_cast<int>((x >> 23) & 0xFF) - 127 + 15;
    std::uint32_t mant = x & 0x7FFFFFu;
    if (exp <= 0) return static_cast<std::uint16_t>(sign);  // flush tiny values
    if (exp >= 31) return static_cast<std::uint16_t>(sign | 0x7C00u);
    std::uint32_t h = sign | (static_cast<std::uint32_t>(exp) << 10) | (mant >> 13);
    const std::uint32_t rest = mant & 0x1FFFu;
    if (rest > 0x1000u || (rest == 0x1000u && (h & 1u))) ++h;
    return static_cast<std::uint16_t>(h);
}

void fill(std::uint16_t* dst, std::size_t n, std::mt19937_64& rng) {
    std::normal_distribution<float> nd(0.f, 1.f);
    for (std::size_t i = 0; i < n; ++i) dst[i] = to_half(nd(rng));
}

}  // namespace

int main(int argc, char** argv) {
    const int L = argc > 1 ? std::atoi(argv[1]) : 4;
    const int B = argc > 2 ? std::atoi(argv[2]) : 64;
    const int H = argc > 3 ? std::atoi(argv[3]) : 32;
    const int s = argc > 4 ? std::atoi(argv[4]) : 512;
    const int steps = argc > 5 ? std::atoi(argv[5]) : 20;
    const int D = 128;
    const double r = 0.2;
    const std::size_t row = static_cast<std::size_t>(B) * H * D;  // one layer's q / k / v [B][H][D]
    try {
        skv::b200::DeviceCache host_path(L, B, H, D, s + steps + 1, SKV_F16, SKV_F16);
        skv::b200::DeviceCache dev_path(L, B, H, D, s + steps + 1, SKV_F16, SKV_F16);
        skv::b200::DeviceCache layer_path(L, B, H, D, s + steps + 1, SKV_F16, SKV_F16);
        std::mt19937_64 rng(2403'17312);
        {  // prompt: s tokens per layer, then the importance seed (engine.hpp:508-512)
            const std::size_t prompt = static_cast<std::size_t>(B) * s * H * D;
            Pinned k(prompt * 2), v(prompt * 2), q(row * 2);
            skv::b200::DeviceBuffer dk(prompt * 2), dv(prompt * 2), dq(row * 2), dout(row * 2);
            for (int l = 0; l < L; ++l) {
                fill(k.as<std::uint16_t>(), prompt, rng);
                fill(v.as<std::uint16_t>(), prompt, rng);
                fill(q.as<std::uint16_t>(), row, rng);
                dk.upload(k.p, prompt * 2);
                dv.upload(v.p, prompt * 2);
                dq.upload(q.p, row * 2);
                for (auto* c : {&host_path, &dev_path, &layer_path}) {
                    c->append_tokens(l, 0, B, 0, s, dk.get(), dv.get());
                    c->prefill_seed(l, s, dq.get(), dout.get());
                }
            }
        }
        const std::size_t step_bytes = static_cast<std::size_t>(L) * row * 2;
        std::vector<Pinned*> qkv;
        for (int j = 0; j < steps; ++j)
            for (int t = 0; t < 3; ++t) {
                qkv.push_back(new Pinned(step_bytes));
                fill(qkv.back()->as<std::uint16_t>(), step_bytes / 2, rng);
            }
        Pinned out_host(step_bytes * steps);
        // host-buffer path, timed: uploads, attention and downloads of every step
        skv::b200::check(skv_stream_synchronize(nullptr));
        const auto t0 = std::chrono::steady_clock::now();
        for (int j = 0; j < steps; ++j)
            host_path.decode_step_host(s + j + 1, r, qkv[3 * j]->p, qkv[3 * j + 1]->p, qkv[3 * j + 2]->p,
                                       out_host.as<std::uint8_t>() + step_bytes * j);
        skv::b200::check(skv_stream_synchronize(nullptr));
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        // layer by layer, synchronous (a host-side model consuming each layer's output)
        std::vector<std::uint8_t> layer_out(step_bytes * steps);
        double sec_layer = 0.0;
        {
            const std::size_t lb = row * 2;
            skv::b200::DeviceBuffer lq(lb), lk(lb), lv(lb), lo(lb);
            const auto t1 = std::chrono::steady_clock::now();
            for (int j = 0; j < steps; ++j)
                for (int l = 0; l < L; ++l) {
                    lq.upload(qkv[3 * j]->as<std::uint8_t>() + lb * l, lb);
                    lk.upload(qkv[3 * j + 1]->as<std::uint8_t>() + lb * l, lb);
                    lv.upload(qkv[3 * j + 2]->as<std::uint8_t>() + lb * l, lb);
                    layer_path.decode_layer(l, s + j + 1, r, lq.get(), lk.get(), lv.get(), lo.get());
                    lo.download(layer_out.data() + step_bytes * j + lb * l, lb);
                }
            sec_layer = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
        }
        int mismatched_layer_steps = 0;
        for (int j = 0; j < steps; ++j)
            if (std::memcmp(layer_out.data() + step_bytes * j, out_host.as<std::uint8_t>() + step_bytes * j,
                            step_bytes) != 0)
                ++mismatched_layer_steps;
        // device-buffer path on the twin cache: must agree bit for bit
        skv::b200::DeviceBuffer dq(step_bytes), dk(step_bytes), dv(step_bytes), dout(step_bytes);
        std::vector<std::uint8_t> got(step_bytes);
        int mismatched_steps = 0;
        for (int j = 0; j < steps; ++j) {
            dq.upload(qkv[3 * j]->p, step_bytes);
            dk.upload(qkv[3 * j + 1]->p, step_bytes);
            dv.upload(qkv[3 * j + 2]->p, step_bytes);
            dev_path.decode_step(s + j + 1, r, dq.get(), dk.get(), dv.get(), dout.get());
            dout.download(got.data(), step_bytes);
            if (std::memcmp(got.data(), out_host.as<std::uint8_t>() + step_bytes * j, step_bytes) != 0)
                ++mismatched_steps;
        }
        const int n = s + steps;
        std::vector<double> ia(static_cast<std::size_t>(B) * n), ib(ia.size());
        int mismatched_layers = 0;
        for (int l = 0; l < L; ++l) {
            host_path.importance(l, 0, B, n, ia.data());
            dev_path.importance(l, 0, B, n, ib.data());
            skv::b200::check(skv_stream_synchronize(nullptr));
            if (ia != ib) ++mismatched_layers;
        }
        for (Pinned* p : qkv) delete p;
        std::printf(
            "{\"program\": \"decode_loop\", \"layers\": %d, \"batch\": %d, \"heads\": %d, \"prompt\": %d, "
            "\"steps\": %d, \"e2e_tokens_per_s\": %.1f, \"e2e_layer_sync_tokens_per_s\": %.1f, "
            "\"mismatched_steps\": %d, \"mismatched_layers\": %d, \"mismatched_layer_sync_steps\": %d}\n",
            L, B, H, s, steps, static_cast<double>(B) * steps / sec, static_cast<double>(B) * steps / sec_layer,
            mismatched_steps, mismatched_layers, mismatched_layer_steps);
        return (mismatched_steps == 0 && mismatched_layers == 0 && mismatched_layer_steps == 0) ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("{\"program\": \"decode_loop\", \"error\": \"%s\"}\n", e.what());
        return 2;
    }
}
