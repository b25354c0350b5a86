// gen_golden.cpp -- emits golden vectors for the W4A8 hot path by running the
// REFERENCE implementation itself (compiled from /root/reference/proj/src by
// oracle/Makefile; never copied into this repo).
//
// TEST INFRASTRUCTURE ONLY.  Output: tests/golden/reference_golden.json, read by
// tests/test_oracle_golden.py (pins the C oracle port) and tests/test_gpu_parity.py
// (pins the CUDA path directly against the reference on the same inputs).
//
// Floats are written as IEEE-754 bit patterns (uint32) so the comparison is
// bit-exact; int8 codes as integers; packed int4 payloads as hex strings.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "core/bench.hpp"
#include "core/clip.hpp"
#include "core/otf.hpp"
#include "core/gemm.hpp"
#include "core/quantize.hpp"
#include "core/rng.hpp"

using namespace ody;

namespace {

std::string out_json;
bool first_case = true;

std::uint32_t bits_of(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

template <typename T>
void emit_int_list(const char* name, const std::vector<T>& v) {
    out_json += "\"";
    out_json += name;
    out_json += "\":[";
    for (std::size_t i = 0; i < v.size(); ++i) {
        if (i) out_json += ",";
        out_json += std::to_string(static_cast<long long>(v[i]));
    }
    out_json += "]";
}

void emit_float_bits(const char* name, const std::vector<float>& v) {
    std::vector<std::uint32_t> b(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) b[i] = bits_of(v[i]);
    emit_int_list(name, b);
}

void emit_hex(const char* name, const std::vector<std::uint8_t>& v) {
    static const char* hx = "0123456789abcdef";
    out_json += "\"";
    out_json += name;
    out_json += "\":\"";
    for (auto b : v) {
        out_json += hx[b >> 4];
        out_json += hx[b & 15];
    }
    out_json += "\"";
}

void begin_case(const std::string& kind, const std::string& name) {
    if (!first_case) out_json += ",\n";
    first_case = false;
    out_json += "{\"kind\":\"" + kind + "\",\"name\":\"" + name + "\",";
}

void end_case() { out_json += "}"; }

QuantScheme per_channel(int bits) {
    QuantScheme s;
    s.bits = bits;
    s.symmetric = true;
    s.granularity = Granularity::PerChannel;
    return s;
}

// One full hot-path case: seeded a ~ N(0,1) (M x K), w ~ sd*N(0,1) (N x K),
// act quant, per-channel W4 quant (optional clip), fast accumulators + output.
void hot_path_case(const std::string& name, std::uint64_t seed, std::size_t m, std::size_t n,
                   std::size_t k, double w_sd, bool with_clip, bool emit_inputs) {
    Rng rng(seed);
    DenseTensor a(m, k);
    for (auto& v : a.data()) v = static_cast<float>(rng.gaussian());
    DenseTensor w(n, k);
    for (auto& v : w.data()) v = static_cast<float>(rng.gaussian() * w_sd);
    QuantScheme sch = per_channel(4);
    if (with_clip) {
        sch.clip_gamma.resize(n);
        sch.clip_beta.resize(n);
        for (std::size_t r = 0; r < n; ++r) {
            sch.clip_gamma[r] = 0.5f + 0.5f * static_cast<float>(rng.uniform());
            sch.clip_beta[r] = 0.5f + 0.5f * static_cast<float>(rng.uniform());
        }
    }
    QuantizedTensor a_q = quantize_activations_per_token(a, 8);
    QuantizedTensor w_q = quantize_weights(w, sch);
    GemmCounters c;
    DenseTensor out = gemm_w4a8_fast(a_q, w_q, &c);
    std::vector<std::int32_t> acc = gemm_w4a8_fast_accumulators(a_q, w_q);

    begin_case("hot_path", name);
    out_json += "\"seed\":" + std::to_string(seed) + ",\"m\":" + std::to_string(m) +
                ",\"n\":" + std::to_string(n) + ",\"k\":" + std::to_string(k) +
                ",\"w_sd\":" + std::to_string(w_sd) + ",\"clip\":" + (with_clip ? "true" : "false") + ",";
    if (emit_inputs && (m * k + n * k) < 20000) {
        emit_float_bits("a_bits", a.data());
        out_json += ",";
        emit_float_bits("w_bits", w.data());
        out_json += ",";
    }
    if (with_clip) {
        emit_float_bits("gamma_bits", sch.clip_gamma);
        out_json += ",";
        emit_float_bits("beta_bits", sch.clip_beta);
        out_json += ",";
    }
    emit_int_list("a_codes", a_q.payload_i8);
    out_json += ",";
    emit_float_bits("a_scales_bits", a_q.scales);
    out_json += ",";
    emit_hex("w_packed", w_q.payload_i4.bytes());
    out_json += ",";
    emit_float_bits("w_scales_bits", w_q.scales);
    out_json += ",";
    emit_int_list("acc16", acc);
    out_json += ",";
    emit_float_bits("out_bits", out.data());
    out_json += ",\"counters\":[" + std::to_string(c.int8_mac_ops) + "," +
                std::to_string(c.dequant_events) + "," + std::to_string(c.zero_point_sub_ops) + "," +
                std::to_string(c.final_scale_ops) + "]";
    end_case();
}

// Bench-style config (bench.cpp:78-113 generator): checksums only, because the
// arrays are large.  FNV-1a (bench.cpp:14-22) over codes, scales, packed
// weights and the f32 output.
void checksum_case(const std::string& name, std::uint64_t seed, std::size_t m, std::size_t n,
                   std::size_t k) {
    Rng rng(seed ^ 0x9d2c5680u);
    DenseTensor a(m, k);
    for (auto& v : a.data()) v = static_cast<float>(rng.gaussian());
    DenseTensor w(n, k);
    for (auto& v : w.data()) v = static_cast<float>(rng.gaussian() * 0.1);
    QuantizedTensor a_q = quantize_activations_per_token(a, 8);
    QuantizedTensor w_q = quantize_weights(w, per_channel(4));
    DenseTensor out = gemm_w4a8_fast(a_q, w_q, nullptr);
    begin_case("checksum", name);
    out_json += "\"seed\":" + std::to_string(seed) + ",\"m\":" + std::to_string(m) +
                ",\"n\":" + std::to_string(n) + ",\"k\":" + std::to_string(k) + ",";
    auto h = [](const void* p, std::size_t b) { return std::to_string(fnv1a(p, b)); };
    out_json += "\"fnv_a_codes\":\"" + h(a_q.payload_i8.data(), a_q.payload_i8.size()) + "\",";
    out_json += "\"fnv_a_scales\":\"" + h(a_q.scales.data(), a_q.scales.size() * 4) + "\",";
    out_json += "\"fnv_w_packed\":\"" + h(w_q.payload_i4.bytes().data(), w_q.payload_i4.bytes().size()) + "\",";
    out_json += "\"fnv_w_scales\":\"" + h(w_q.scales.data(), w_q.scales.size() * 4) + "\",";
    out_json += "\"fnv_out\":\"" + h(out.data().data(), out.data().size() * 4) + "\",";
    std::vector<float> head(out.data().begin(), out.data().begin() + std::min<std::size_t>(16, out.size()));
    emit_float_bits("out_head_bits", head);
    end_case();
}

// The comparison engines (gemm.cpp:105-311) on one seeded input: f32 outputs + counters.
// w8a8: 8-bit per-channel weights; finegrained: 4-bit per-group (group g); asymmetric:
// run_engine's uint4-offset path over the per-channel 4-bit codes; w4a16: per-group
// 4-bit weights against the dense activations.
void engine_case(const std::string& name, std::uint64_t seed, std::size_t m, std::size_t n, std::size_t k,
                 std::size_t g) {
    Rng rng(seed);
    DenseTensor a(m, k);
    for (auto& v : a.data()) v = static_cast<float>(rng.gaussian());
    DenseTensor w(n, k);
    for (auto& v : w.data()) v = static_cast<float>(rng.gaussian() * 0.1);
    QuantizedTensor a_q = quantize_activations_per_token(a, 8);
    QuantizedTensor w4 = quantize_weights(w, per_channel(4));
    QuantizedTensor w8 = quantize_weights(w, per_channel(8));
    QuantScheme grp = per_channel(4);
    grp.granularity = Granularity::PerGroup;
    grp.group_size = g;
    QuantizedTensor wg = quantize_weights(w, grp);
    begin_case("engines", name);
    out_json += "\"seed\":" + std::to_string(seed) + ",\"m\":" + std::to_string(m) + ",\"n\":" +
                std::to_string(n) + ",\"k\":" + std::to_string(k) + ",\"group\":" + std::to_string(g) + ",";
    emit_int_list("w8_codes", w8.payload_i8);
    out_json += ",";
    emit_float_bits("w8_scales_bits", w8.scales);
    out_json += ",";
    emit_hex("wg_packed", wg.payload_i4.bytes());
    out_json += ",";
    emit_float_bits("wg_scales_bits", wg.scales);
    struct E {
        const char* key;
        Engine e;
        const QuantizedTensor* wq;
    } es[] = {{"w8a8", Engine::W8A8, &w8},
              {"finegrained", Engine::W4A8FineGrained, &wg},
              {"asymmetric", Engine::W4A8Asymmetric, &w4},
              {"fast", Engine::W4A8Fast, &w4},
              {"w4a16", Engine::W4A16Grouped, &wg}};
    for (const E& e : es) {
        GemmCounters c;
        DenseTensor out = run_engine(e.e, a, a_q, *e.wq, &c);
        out_json += ",";
        emit_float_bits((std::string(e.key) + "_out_bits").c_str(), out.data());
        out_json += ",\"" + std::string(e.key) + "_counters\":[" + std::to_string(c.int8_mac_ops) + "," +
                    std::to_string(c.dequant_events) + "," + std::to_string(c.zero_point_sub_ops) + "," +
                    std::to_string(c.final_scale_ops) + "]";
    }
    end_case();
}

// LWC grid search (clip.cpp:55-103) on a seeded weight, grid (0.5, 0.01) and (0.3, 0.07).
void lwc_case(const std::string& name, std::uint64_t seed, std::size_t n, std::size_t k, int bits, float gmin,
              float gstep) {
    Rng rng(seed);
    DenseTensor w(n, k);
    for (auto& v : w.data()) v = static_cast<float>(rng.gaussian() * 0.1);
    if (n > 2) {  // an outlier channel and an all-zero channel
        w.at(1, 0) = 3.0f;
        for (std::size_t c = 0; c < k; ++c) w.at(2, c) = 0.0f;
    }
    ClipResult r = optimize_clipping(w, bits, ClipGrid{gmin, gstep});
    begin_case("lwc", name);
    out_json += "\"seed\":" + std::to_string(seed) + ",\"n\":" + std::to_string(n) + ",\"k\":" +
                std::to_string(k) + ",\"bits\":" + std::to_string(bits) + ",\"gmin_bits\":" +
                std::to_string(bits_of(gmin)) + ",\"gstep_bits\":" + std::to_string(bits_of(gstep)) + ",";
    emit_float_bits("w_bits", w.data());
    out_json += ",";
    emit_float_bits("gamma_bits", r.gamma);
    out_json += ",";
    emit_float_bits("beta_bits", r.beta);
    out_json += ",";
    emit_float_bits("mse_before_bits", r.mse_before);
    out_json += ",";
    emit_float_bits("mse_after_bits", r.mse_after);
    end_case();
}

// The OTF bytes write_tensor (otf.cpp:121-153) produces for a small 4-bit tensor.
void otf_case() {
    Rng rng(4242);
    DenseTensor w(3, 5);
    for (auto& v : w.data()) v = static_cast<float>(rng.gaussian() * 0.1);
    QuantizedTensor q = quantize_weights(w, per_channel(4));
    const std::string dir = "/tmp/ody_golden_otf";
    write_tensor(q, dir);
    auto slurp = [](const std::string& p) {
        std::vector<std::uint8_t> b;
        FILE* f = std::fopen(p.c_str(), "rb");
        int c;
        while (f && (c = std::fgetc(f)) != EOF) b.push_back(static_cast<std::uint8_t>(c));
        if (f) std::fclose(f);
        return b;
    };
    begin_case("otf", "w4_3x5");
    emit_float_bits("w_bits", w.data());
    out_json += ",";
    emit_hex("payload_otf", slurp(dir + "/payload.otf"));
    out_json += ",";
    emit_hex("scales_otf", slurp(dir + "/scales.otf"));
    out_json += ",";
    emit_hex("scheme_txt", slurp(dir + "/scheme.txt"));
    end_case();
}

} // namespace

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "reference_golden.json";
    out_json = "{\"generator\":\"oracle/gen_golden.cpp against /root/reference/proj/src\",\"cases\":[\n";

    // Known-answer scalar cases from proj/tests/test_quantizer.cpp:9-42,108-119.
    {
        std::vector<float> w{0.4f, -0.2f, 0.1f};
        SymmetricQuant q = quantize_symmetric(w, 4, 1.0f, 1.0f);
        begin_case("symmetric", "w3_bits4");
        emit_float_bits("x_bits", w);
        out_json += ",\"bits\":4,\"gamma_bits\":" + std::to_string(bits_of(1.0f)) +
                    ",\"beta_bits\":" + std::to_string(bits_of(1.0f)) + ",";
        emit_int_list("codes", q.codes);
        out_json += ",\"scale_bits\":" + std::to_string(bits_of(q.scale));
        end_case();
        std::vector<float> clip{0.4f, -0.4f};
        SymmetricQuant qc = quantize_symmetric(clip, 4, 0.5f, 0.5f);
        begin_case("symmetric", "clip_half_bits4");
        emit_float_bits("x_bits", clip);
        out_json += ",\"bits\":4,\"gamma_bits\":" + std::to_string(bits_of(0.5f)) +
                    ",\"beta_bits\":" + std::to_string(bits_of(0.5f)) + ",";
        emit_int_list("codes", qc.codes);
        out_json += ",\"scale_bits\":" + std::to_string(bits_of(qc.scale));
        end_case();
        std::vector<float> r127{1.27f, 1.27f, 1.27f};
        SymmetricQuant q8 = quantize_symmetric(r127, 8, 1.0f, 1.0f);
        begin_case("symmetric", "row_1p27_bits8");
        emit_float_bits("x_bits", r127);
        out_json += ",\"bits\":8,\"gamma_bits\":" + std::to_string(bits_of(1.0f)) +
                    ",\"beta_bits\":" + std::to_string(bits_of(1.0f)) + ",";
        emit_int_list("codes", q8.codes);
        out_json += ",\"scale_bits\":" + std::to_string(bits_of(q8.scale));
        end_case();
        std::vector<float> z{0.0f, 0.0f, 0.0f, 0.0f};
        SymmetricQuant qz = quantize_symmetric(z, 8, 1.0f, 1.0f);
        begin_case("symmetric", "zero_row_bits8");
        emit_float_bits("x_bits", z);
        out_json += ",\"bits\":8,\"gamma_bits\":" + std::to_string(bits_of(1.0f)) +
                    ",\"beta_bits\":" + std::to_string(bits_of(1.0f)) + ",";
        emit_int_list("codes", qz.codes);
        out_json += ",\"scale_bits\":" + std::to_string(bits_of(qz.scale));
        end_case();
    }

    // The run_verify random-matrix sweep shapes (pipeline.cpp:186-230): 20 seeded
    // (m,n,k) in [1,64], inputs included so the GPU path can replay them.
    {
        Rng shape_rng(1);
        for (int trial = 0; trial < 20; ++trial) {
            std::size_t m = static_cast<std::size_t>(shape_rng.uniform_int(1, 64));
            std::size_t n = static_cast<std::size_t>(shape_rng.uniform_int(1, 64));
            std::size_t k = static_cast<std::size_t>(shape_rng.uniform_int(1, 64));
            hot_path_case("verify_trial_" + std::to_string(trial), 1000 + trial, m, n, k, 0.1,
                          trial % 5 == 3, true);
        }
    }
    // Ragged / edge shapes: K odd, M=1, N=1, K=1, K not a multiple of 128.
    hot_path_case("edge_k1", 7, 3, 5, 1, 0.3, false, true);
    hot_path_case("edge_m1_n1", 8, 1, 1, 37, 0.3, false, true);
    hot_path_case("edge_k129", 9, 5, 7, 129, 0.1, false, true);
    hot_path_case("edge_n130_k200", 10, 2, 130, 200, 0.1, true, true);
    hot_path_case("mid_m17_n257_k384", 11, 17, 257, 384, 0.1, false, true);

    // Bench-generator checksums (bench.cpp:78-113), seed 1.
    checksum_case("cfg1_m16_n4096_k4096", 1, 16, 4096, 4096);
    checksum_case("o_m1_n5120_k5120", 1, 1, 5120, 5120);
    checksum_case("mixed_m64_n384_k5120", 1, 64, 384, 5120);

    // Comparison engines and the LWC grid search (row 4).
    engine_case("engines_m5_n40_k64_g16", 501, 5, 40, 64, 16);
    engine_case("engines_m16_n130_k384_g128", 502, 16, 130, 384, 128);
    engine_case("engines_m3_n7_k96_g32", 503, 3, 7, 96, 32);
    lwc_case("lwc_n6_k64_b4", 601, 6, 64, 4, 0.5f, 0.01f);
    lwc_case("lwc_n5_k300_b4_coarse", 602, 5, 300, 4, 0.3f, 0.07f);
    lwc_case("lwc_n4_k128_b8", 603, 4, 128, 8, 0.5f, 0.01f);
    otf_case();

    out_json += "\n]}\n";
    FILE* f = std::fopen(path, "w");
    if (!f) return 2;
    std::fwrite(out_json.data(), 1, out_json.size(), f);
    std::fclose(f);
    std::printf("wrote %s (%zu bytes)\n", path, out_json.size());
    return 0;
}
