// examples/train_window.cpp — a C++ host driving the snake progression
// through the C-ABI exactly as the reference trainer loop would:
// for each window position, n_it iterations of train_step, then a run
// checkpoint and a PSNR of the view's crop.  Builds against include/ and
// links libtilefield_gpu.so.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <string>
#include <vector>

#include "../include/tilefield_gpu.hpp"

int main() {
    tfg_field_config f;
    tfg_train_config t;
    tfg_default_field_config(&f);
    tfg_default_train_config(&t);
    t.batch_rays = 4096;
    // a 3x3 grid of 128 m tiles seen by one nadir camera (affine RPC)
    tfg_roi roi{0, 384, 0, 384, 0, 40};
    tfg_rpc cam{};
    cam.long_off = cam.lat_off = 192;
    cam.height_off = 20;
    cam.long_scale = cam.lat_scale = 211;
    cam.height_scale = 24;
    cam.samp_scale = cam.line_scale = 211 / 0.5;
    cam.samp_off = cam.line_off = 400;
    cam.samp_num[1] = 1;
    cam.line_num[2] = -1;
    cam.samp_den[0] = cam.line_den[0] = 1;
    cam.image_rows = cam.image_cols = 800;
    std::vector<uint8_t> img(800 * 800 * 3);
    for (size_t i = 0; i < img.size(); ++i) img[i] = uint8_t((i * 2654435761u) >> 24);
    try {
        tilefield::gpu::Context ctx(f, t, 0, 4096);
        ctx.set_scene({cam}, {img.data()}, roi, 3, 3);
        uint64_t it = 0;
        for (auto [r, c] : tilefield::gpu::Context::snake_path(3, 3)) {
            ctx.advance(r, c);
            float loss = 0;
            for (int k = 0; k < 8; ++k) loss = ctx.train_step(it++, 0, 4096);
            std::printf("window (%d,%d): %llu accepted rays, loss %.5f\n", r, c,
                        (unsigned long long)ctx.accepted_rays(), loss);
        }
        // run checkpoint (tiles/r{R}_c{C}.ckpt + color_net.ckpt)
        std::string dir = std::string(std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp") + "/tfg_example_run";
        std::filesystem::create_directories(dir + "/tiles");
        ctx.save_run(dir);
        // evaluation metric on the GPU: PSNR of the image against a shifted copy
        std::vector<float> a(64 * 64 * 3), b(a.size());
        for (size_t i = 0; i < a.size(); ++i) {
            a[i] = img[i] / 255.f;
            b[i] = std::fmin(1.f, a[i] + 0.1f);
        }
        std::printf("checkpointed to %s; psnr %.2f dB\n", dir.c_str(), ctx.psnr(a.data(), b.data(), a.size()));
    } catch (const tilefield::Error& e) {
        std::printf("tilefield::Error: %s\n", e.what());
        return 1;
    }
    return 0;
}
