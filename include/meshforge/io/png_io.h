// meshforge PNG I/O (source-compatible with proj/include/meshforge/io/png_io.h),
// written directly over zlib (the reference's libpng is not needed): 8-bit
// gray / RGB; alpha stripped on read; encode filters rows adaptively and
// deflates row bands on all host threads (independent pigz-style blocks).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "meshforge/core/image.h"

namespace meshforge {

ImageU8 readPng(const std::string& path);
void writePng(const std::string& path, const ImageU8& image);

std::vector<std::uint8_t> encodePng(const ImageU8& image);
ImageU8 decodePng(const std::uint8_t* bytes, std::size_t size);

}  // namespace meshforge
