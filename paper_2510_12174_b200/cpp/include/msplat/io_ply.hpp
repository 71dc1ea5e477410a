// msplat C++ drop-in -- extended-PLY I/O (reference API:
// proj/core/include/msplat/io_ply.hpp).  Scene files are decoded / encoded on
// the device (msplat_load_scene_ply / msplat_save_scene_ply); the plain point
// cloud files are host I/O.
#pragma once

#include "msplat/scene.hpp"

#include <string>
#include <vector>

namespace msplat {

void save_scene_ply(const std::string& path, const Scene& scene);
Scene load_scene_ply(const std::string& path);

void save_points_ply(const std::string& path, const std::vector<Vec3>& points, const std::vector<Vec3>& colors);
void load_points_ply(const std::string& path, std::vector<Vec3>& points, std::vector<Vec3>& colors);

}  // namespace msplat
