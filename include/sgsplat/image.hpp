// sgsplat/image.hpp -- H x W x C row-major double image (drop-in declarations).
// Mirrors proj/include/sgsplat/image.hpp:12-43 (PNG / FIMG file I/O is out of scope).
#pragma once

#include <cstddef>
#include <vector>

namespace sgsplat {

struct Image {
    int width = 0;
    int height = 0;
    int channels = 3;
    std::vector<double> data;

    Image() = default;
    Image(int w, int h, int c = 3)
        : width(w), height(h), channels(c),
          data(static_cast<std::size_t>(w) * static_cast<std::size_t>(h) * static_cast<std::size_t>(c), 0.0) {}

    std::size_t index(int y, int x, int c) const {
        return (static_cast<std::size_t>(y) * static_cast<std::size_t>(width) + static_cast<std::size_t>(x)) *
                   static_cast<std::size_t>(channels) +
               static_cast<std::size_t>(c);
    }
    double& at(int y, int x, int c) { return data[index(y, x, c)]; }
    double at(int y, int x, int c) const { return data[index(y, x, c)]; }
    std::size_t size() const { return data.size(); }
    bool same_shape(const Image& o) const {
        return width == o.width && height == o.height && channels == o.channels;
    }
    Image clamped01() const;
};

}  // namespace sgsplat
