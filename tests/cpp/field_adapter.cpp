// field_adapter.cpp — a reference-style caller of the drop-in batch operators
// (include/tilefield_gpu_field.hpp: forward_batch / backward_batch / adam_step
// with the field.hpp:45-48,185-197 signatures).  tests/test_gpu_adapter.py
// writes a caller-built RaySegmentBatch (the CPU oracle's), the tile / colour
// parameters and d_sigma / d_rgb as raw little-endian files into a directory;
// this program runs the three operators on the GPU through the C-ABI and
// writes sigma, rgb, the gradients and the Adam-updated colour state back.
//
//   field_adapter <dir>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "tilefield_gpu_field.hpp"

template <typename T>
static std::vector<T> load(const std::string& path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw tilefield::Error("cannot open " + path);
    const size_t n = size_t(f.tellg()) / sizeof(T);
    std::vector<T> v(n);
    f.seekg(0);
    f.read(reinterpret_cast<char*>(v.data()), std::streamsize(n * sizeof(T)));
    return v;
}
template <typename T>
static void save(const std::string& path, const std::vector<T>& v) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(T)));
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: field_adapter <dir>\n");
        return 2;
    }
    const std::string d = argv[1];
    try {
        using namespace tilefield;
        // the caller's batch (RaySegmentBatch, ray_batch.hpp:13-49)
        const auto rays = load<tfg_ray_entry>(d + "/rays.bin");
        RaySegmentBatch batch;
        batch.rays.resize(rays.size());
        for (size_t i = 0; i < rays.size(); ++i) {
            auto& r = batch.rays[i];
            for (int q = 0; q < 3; ++q) {
                r.origin[q] = rays[i].origin[q];
                r.direction[q] = rays[i].direction[q];
                r.target[q] = rays[i].target[q];
            }
            r.image_id = rays[i].image_id;
            r.pixel.row = rays[i].row;
            r.pixel.col = rays[i].col;
        }
        batch.offsets = load<uint32_t>(d + "/offsets.bin");
        batch.t = load<float>(d + "/t.bin");
        batch.delta = load<float>(d + "/delta.bin");
        batch.local = load<float>(d + "/local.bin");
        batch.slot = load<uint8_t>(d + "/slot.bin");
        batch.endpoint = load<uint8_t>(d + "/endpoint.bin");
        // the caller's parameters (TileField / GlobalColorNet storage)
        std::vector<std::vector<float>> enc(4), dnet(4);
        for (int k = 0; k < 4; ++k) {
            enc[k] = load<float>(d + "/enc" + std::to_string(k) + ".bin");
            dnet[k] = load<float>(d + "/dnet" + std::to_string(k) + ".bin");
        }
        std::vector<float> color = load<float>(d + "/color.bin");
        tfg_field_config fc{};
        tfg_train_config tc{};
        tfg_default_field_config(&fc);
        tfg_default_train_config(&tc);
        gpu::Context ctx(fc, tc, 0, int(batch.rays.size()));
        gpu::set_default_context(&ctx);
        std::vector<FieldParamView<float>> views(4);
        for (int k = 0; k < 4; ++k) {
            views[k].cfg = &fc;
            views[k].enc_tables = enc[k].data();
            views[k].dnet_params = dnet[k].data();
        }
        ColorParamView<float> cv;
        cv.cfg = &fc;
        cv.params = color.data();
        ForwardWorkspace<float> ws;
        gpu::forward_batch<float>(batch, std::span<const FieldParamView<float>>(views), cv, ws, 8);
        save(d + "/out_sigma.bin", ws.sigma);
        save(d + "/out_rgb.bin", ws.rgb);
        const auto ds = load<float>(d + "/d_sigma.bin");
        const auto dr = load<float>(d + "/d_rgb.bin");
        BatchGrads<float> grads;
        gpu::backward_batch<float>(batch, std::span<const FieldParamView<float>>(views), cv, ws,
                                   std::span<const float>(ds), std::span<const float>(dr), grads, 8);
        for (int k = 0; k < 4; ++k) {
            save(d + "/out_genc" + std::to_string(k) + ".bin", grads.tiles[k].enc);
            save(d + "/out_gdnet" + std::to_string(k) + ".bin", grads.tiles[k].dnet);
        }
        save(d + "/out_gcolor.bin", grads.color);
        // adam_step on the colour group with the computed gradient
        AdamState st;
        st.m = load<float>(d + "/adam_m.bin");
        st.v = load<float>(d + "/adam_v.bin");
        st.step = 7;
        LrSchedule sched;
        sched.base = 1e-3;
        AdamConfig acfg;
        std::vector<float> p = color;
        gpu::adam_step(std::span<float>(p), std::span<const float>(grads.color), st, sched, acfg, "color");
        save(d + "/out_adam_p.bin", p);
        save(d + "/out_adam_m.bin", st.m);
        save(d + "/out_adam_v.bin", st.v);
        std::vector<uint64_t> step{st.step};
        save(d + "/out_adam_step.bin", step);
        // the error contract: a non-finite gradient throws naming the group
        std::vector<float> bad = grads.color;
        bad[3] = std::nanf("");
        try {
            gpu::adam_step(std::span<float>(p), std::span<const float>(bad), st, sched, acfg, "color");
            std::fprintf(stderr, "adam_step accepted a NaN gradient\n");
            return 1;
        } catch (const Error& e) {
            std::printf("expected error: %s\n", e.what());
        }
        std::printf("ok %zu rays %zu samples\n", batch.rays.size(), batch.t.size());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
