// Flat C entry points over the reference's own dataset / image / config I/O
// (core/src/dataset.cpp, core/src/io_image.cpp, compiled unmodified into
// _ref/libmsplat_ref_io.so with nlohmann/json from the image and libpng16 from
// Pillow's wheel through pngshim/png.h).  The same shapes as the drop-in's
// msplat_dataset_* / msplat_image_* / msplat_config_load, so a test can call
// both and compare.  TEST INFRASTRUCTURE ONLY.
#include "msplat/dataset.hpp"
#include "msplat/io_image.hpp"
#include "msplat/trainer.hpp"

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

namespace {
thread_local std::string g_err;
}

#define MO_EXPORT extern "C" __attribute__((visibility("default")))

MO_EXPORT const char* mo_io_last_error() { return g_err.c_str(); }

MO_EXPORT int mo_io_dataset_load(const char* root, void** out) {
    try {
        *out = new msplat::SceneDataset(msplat::load_dataset(root));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        *out = nullptr;
        return 1;
    }
}

MO_EXPORT void mo_io_dataset_free(void* h) { delete static_cast<msplat::SceneDataset*>(h); }

MO_EXPORT void mo_io_dataset_dims(void* h, int64_t dims[5]) {
    const auto* ds = static_cast<const msplat::SceneDataset*>(h);
    dims[0] = ds->width;
    dims[1] = ds->height;
    dims[2] = ds->num_classes;
    dims[3] = int64_t(ds->frames.size());
    dims[4] = int64_t(ds->points.size());
}

MO_EXPORT int mo_io_dataset_frame(void* h, int64_t i, double cam[16], int* flags, float* rgb, float* depth,
                                  float* normal, uint8_t* labels) {
    const auto* ds = static_cast<const msplat::SceneDataset*>(h);
    if (i < 0 || i >= int64_t(ds->frames.size())) return 1;
    const auto& f = ds->frames[size_t(i)];
    const auto& v = f.view;
    cam[0] = v.fx;
    cam[1] = v.fy;
    cam[2] = v.cx;
    cam[3] = v.cy;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) cam[4 + r * 3 + c] = v.R_cam_to_world(r, c);
    for (int k = 0; k < 3; ++k) cam[13 + k] = v.t_cam_to_world[k];
    *flags = (f.rgb.empty() ? 0 : 1) | (f.depth.empty() ? 0 : 2) | (f.normal.empty() ? 0 : 4) |
             (f.labels.empty() ? 0 : 8) | (f.split == "test" ? 16 : 0);
    const size_t HW = size_t(ds->width) * ds->height;
    auto planar = [&](const msplat::GridF& g, float* dst) {
        if (!dst || g.empty()) return;
        const int C = g.channels();
        for (size_t p = 0; p < HW; ++p)
            for (int c = 0; c < C; ++c) dst[size_t(c) * HW + p] = float(g.storage()[p * C + c]);
    };
    planar(f.rgb, rgb);
    planar(f.depth, depth);
    planar(f.normal, normal);
    if (labels && !f.labels.empty()) std::memcpy(labels, f.labels.storage().data(), HW);
    return 0;
}

MO_EXPORT void mo_io_dataset_points(void* h, double* points, double* colors) {
    const auto* ds = static_cast<const msplat::SceneDataset*>(h);
    for (size_t i = 0; i < ds->points.size(); ++i)
        for (int k = 0; k < 3; ++k) {
            if (points) points[i * 3 + k] = ds->points[i][k];
            if (colors) colors[i * 3 + k] = i < ds->point_colors.size() ? ds->point_colors[i][k] : 0.0;
        }
}

MO_EXPORT int mo_io_dataset_save(void* h, const char* root) {
    try {
        msplat::save_dataset(root, *static_cast<const msplat::SceneDataset*>(h));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

MO_EXPORT int mo_io_read_png(const char* path, int* w, int* h, int* c, uint8_t* out) {
    try {
        const msplat::GridU8 g = msplat::read_png(path);
        *w = g.width();
        *h = g.height();
        *c = g.channels();
        if (out) std::memcpy(out, g.storage().data(), g.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

MO_EXPORT int mo_io_write_png(const char* path, int w, int h, int c, const uint8_t* in) {
    try {
        msplat::GridU8 g(w, h, c);
        std::memcpy(g.storage().data(), in, g.size());
        msplat::write_png(path, g);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

MO_EXPORT int mo_io_read_pfm(const char* path, int* w, int* h, int* c, double* out) {
    try {
        const msplat::GridF g = msplat::read_pfm(path);
        *w = g.width();
        *h = g.height();
        *c = g.channels();
        if (out) std::memcpy(out, g.storage().data(), g.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

MO_EXPORT int mo_io_write_pfm(const char* path, int w, int h, int c, const double* in) {
    try {
        msplat::GridF g(w, h, c);
        std::memcpy(g.storage().data(), in, g.size() * sizeof(double));
        msplat::write_pfm(path, g);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

MO_EXPORT int mo_io_config_load(const char* path, double out[33]) {
    try {
        const msplat::TrainConfig c = msplat::load_config(path);
        const double v[33] = {double(c.iterations), c.lr_position, c.lr_rotation, c.lr_scale, c.lr_opacity, c.lr_sh,
                              c.lr_semantics, c.lr_k, c.lambdas[0], c.lambdas[1], c.lambdas[2], c.lambdas[3],
                              c.lambdas[4], c.lambdas[5], double(c.prune_interval), c.prune_threshold,
                              double(c.prune_enabled), double(c.prune_keep_small), c.k_reset, double(c.step1),
                              double(c.step2), c.lambda_fuse, c.mask_threshold, c.sigma_scale,
                              c.early_stop_transmittance, c.background[0], c.background[1], c.background[2],
                              double(c.sh_degree), double(c.seed), double(c.threads), double(c.deterministic)};
        std::memcpy(out, v, sizeof(v));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
