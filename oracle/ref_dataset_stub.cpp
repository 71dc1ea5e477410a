// Link stub for the two SceneDataset members trainer.cpp references
// (core/src/dataset.cpp:19-33).  dataset.cpp itself is not compiled into the
// oracle because it drags in nlohmann/json, libpng and PLY I/O, none of which
// are on the rasterizer hot path.  The split
// rule restated here is the reference's: frames whose split is not "test" /
// is "test", in index order.  TEST INFRASTRUCTURE ONLY.
#include "msplat/dataset.hpp"

namespace msplat {

std::vector<int> SceneDataset::train_indices() const {
    std::vector<int> out;
    for (int i = 0; i < int(frames.size()); ++i)
        if (frames[i].split != "test")
            out.push_back(i);
    return out;
}

std::vector<int> SceneDataset::test_indices() const {
    std::vector<int> out;
    for (int i = 0; i < int(frames.size()); ++i)
        if (frames[i].split == "test")
            out.push_back(i);
    return out;
}

} // namespace msplat
