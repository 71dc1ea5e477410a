/* Host-side dataset / image / config I/O of the C++ drop-in
 * (paper_2510_12174_b200/libmsplat_dropin.so, src/dataset_io.cpp).
 *
 * These are the flat entry points a binding of the reference's
 *   msplat::load_dataset / save_dataset / load_config   (core/src/dataset.cpp:53-284)
 *   msplat::read_png / write_png / read_pfm / write_pfm (core/src/io_image.cpp:28-171)
 * would call: the files are parsed and decoded on the host (as in the
 * reference), and msplat_dataset_frame hands the maps back planar so they go
 * to the device unchanged as msplat_ground_truth (msplat_b200.h).
 * Status: 0 = ok, 1 = error with the reference's message in
 * msplat_dataset_last_error() (thread-local). */
#ifndef MSPLAT_IO_H
#define MSPLAT_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSPLAT_IO_API __attribute__((visibility("default")))

MSPLAT_IO_API const char* msplat_dataset_last_error(void);

/* load_dataset (dataset.cpp:53-145) into an opaque handle. */
MSPLAT_IO_API int msplat_dataset_load(const char* root, void** out);
MSPLAT_IO_API void msplat_dataset_free(void* dataset);
/* dims = {width, height, num_classes, frames, points} */
MSPLAT_IO_API void msplat_dataset_dims(void* dataset, int64_t dims[5]);
/* cam = {fx, fy, cx, cy, R_c2w[9] row-major, t_c2w[3]}; flags bit0 rgb, bit1 depth,
 * bit2 normal, bit3 labels, bit4 split == "test".  Present maps are written
 * planar: rgb [3][H][W], depth [H][W], normal [3][H][W] (float), labels [H][W]
 * (uint8).  Any output pointer may be NULL. */
MSPLAT_IO_API int msplat_dataset_frame(void* dataset, int64_t index, double cam[16], int* flags, float* rgb,
                                       float* depth, float* normal, uint8_t* labels);
/* points / colors: [points][3] doubles (colors in [0, 1]); either may be NULL. */
MSPLAT_IO_API void msplat_dataset_points(void* dataset, double* points, double* colors);
/* save_dataset (dataset.cpp:147-208) of a loaded dataset under `root`. */
MSPLAT_IO_API int msplat_dataset_save(void* dataset, const char* root);

/* read_png / write_png (io_image.cpp:92-171): pixel-major [H][W][C] bytes,
 * C = 1 or 3.  Reading with out == NULL returns the shape only. */
MSPLAT_IO_API int msplat_image_read_png(const char* path, int* width, int* height, int* channels, uint8_t* out);
MSPLAT_IO_API int msplat_image_write_png(const char* path, int width, int height, int channels, const uint8_t* in);
/* read_pfm / write_pfm (io_image.cpp:28-90): [H][W][C] doubles, C = 1 or 3. */
MSPLAT_IO_API int msplat_image_read_pfm(const char* path, int* width, int* height, int* channels, double* out);
MSPLAT_IO_API int msplat_image_write_pfm(const char* path, int width, int height, int channels, const double* in);

/* load_config (dataset.cpp:210-284) into 33 doubles: iterations,
 * lr_{position,rotation,scale,opacity,sh,semantics,k}, lambdas[6],
 * prune_interval, prune_threshold, prune_enabled, prune_keep_small, k_reset,
 * step1, step2, lambda_fuse, mask_threshold, sigma_scale,
 * early_stop_transmittance, background[3], sh_degree, seed, threads,
 * deterministic. */
MSPLAT_IO_API int msplat_config_load(const char* path, double out[33]);

#ifdef __cplusplus
}
#endif

#endif /* MSPLAT_IO_H */
