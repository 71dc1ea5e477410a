// Times the C++ drop-in (libmsplat_dropin.so) at the reference's own API
// boundary (proj/core/include/msplat/rasterizer.hpp:67-83): msplat::rasterize
// and msplat::rasterize_backward with the scene, frame, replay and gradients as
// host Eigen / AoS data -- every call marshals host <-> device, exactly what a
// reference user who relinks against the drop-in gets.
//
//   dropin_bench <scene.ply> <fx> <fy> <cx> <cy> <W> <H> <R00..R22 (9)> <t0 t1 t2> <warmup> <iters>
//
// Precision / determinism follow the drop-in's environment switches
// (MSPLAT_PRECISION=32, MSPLAT_DETERMINISTIC=0).  Prints one JSON object:
// per-iteration wall-clock of rasterize, rasterize_backward and their sum.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "msplat/io_ply.hpp"
#include "msplat/rasterizer.hpp"

using namespace msplat;

int main(int argc, char** argv) {
    if (argc != 1 + 7 + 9 + 3 + 2) {
        std::fprintf(stderr, "usage: dropin_bench scene.ply fx fy cx cy W H R(9) t(3) warmup iters\n");
        return 2;
    }
    int i = 1;
    const std::string path = argv[i++];
    const double fx = std::atof(argv[i++]), fy = std::atof(argv[i++]);
    const double cx = std::atof(argv[i++]), cy = std::atof(argv[i++]);
    const int W = std::atoi(argv[i++]), H = std::atoi(argv[i++]);
    Mat3 R;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) R(r, c) = std::atof(argv[i++]);
    Vec3 t;
    for (int r = 0; r < 3; ++r) t[r] = std::atof(argv[i++]);
    const int warmup = std::atoi(argv[i++]), iters = std::atoi(argv[i++]);

    const Scene scene = load_scene_ply(path);
    const CameraView view = make_camera(fx, fy, cx, cy, W, H, R, t);
    RenderConfig cfg;
    cfg.background = Vec3(0.1, 0.2, 0.3);
    const int C = scene.num_classes;
    // dense synthetic pixel gradients, U(-1, 1) / (W H) as in bench.py
    PixelGradients pix = PixelGradients::zero(W, H, C);
    std::mt19937_64 rng(4);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    const double s = 1.0 / (double(W) * H);
    for (GridF* g : {&pix.dcolor, &pix.ddepth, &pix.dsemantics, &pix.dkmap})
        for (size_t k = 0; k < g->size(); ++k) g->data()[k] = u(rng) * s;

    using clk = std::chrono::steady_clock;
    double fwd = 0, bwd = 0;
    double checksum = 0;
    for (int it = 0; it < warmup + iters; ++it) {
        ReplayState replay;
        const auto t0 = clk::now();
        const MultimodalFrame frame = rasterize(scene, view, cfg, &replay);
        const auto t1 = clk::now();
        const GradientBuffer g = rasterize_backward(scene, view, frame, replay, pix);
        const auto t2 = clk::now();
        if (it >= warmup) {
            fwd += std::chrono::duration<double, std::milli>(t1 - t0).count();
            bwd += std::chrono::duration<double, std::milli>(t2 - t1).count();
        }
        checksum = frame.color.data()[0] + g.dopacity[0];
    }
    const char* prec = std::getenv("MSPLAT_PRECISION");
    const char* det = std::getenv("MSPLAT_DETERMINISTIC");
    std::printf("{\"n\": %zu, \"width\": %d, \"height\": %d, \"classes\": %d, \"precision\": \"%s\", "
                "\"deterministic\": %s, \"iters\": %d, \"rasterize_ms\": %.3f, \"rasterize_backward_ms\": %.3f, "
                "\"fwd_bwd_ms\": %.3f, \"renders_per_s\": %.3f, \"checksum\": %.6e}\n",
                scene.size(), W, H, C, (prec && std::string(prec) == "32") ? "f32" : "f64",
                (det && std::string(det) == "0") ? "false" : "true", iters, fwd / iters, bwd / iters,
                (fwd + bwd) / iters, 1000.0 * iters / (fwd + bwd), checksum);
    return 0;
}
