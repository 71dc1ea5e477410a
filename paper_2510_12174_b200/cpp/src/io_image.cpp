// Ground-truth image I/O for the C++ drop-in (reference: core/src/io_image.cpp).
//   PFM   io_image.cpp:28-90   (same header, bottom-up rows, endian marker)
//   PNG   io_image.cpp:92-171  (libpng there; zlib + the PNG spec here)
//   to_u8 / to_unit            io_image.cpp:173-187
// Error texts are the reference's ("<path>: <what>").
#include "msplat/io_image.hpp"

#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

namespace msplat {

namespace {

[[noreturn]] void fail(const std::string& path, const std::string& msg) {
    throw std::runtime_error(path + ": " + msg);
}

bool host_little_endian() {
    const uint32_t probe = 1;
    uint8_t b;
    std::memcpy(&b, &probe, 1);
    return b == 1;
}

const uint8_t kPngSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};

uint32_t be32(const uint8_t* p) { return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3]; }
void put_be32(std::vector<uint8_t>& out, uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) out.push_back(uint8_t(v >> s));
}

void put_chunk(std::vector<uint8_t>& out, const char* type, const uint8_t* data, size_t n) {
    put_be32(out, uint32_t(n));
    const size_t at = out.size();
    out.insert(out.end(), type, type + 4);
    if (n) out.insert(out.end(), data, data + n);
    uLong crc = crc32(0L, Z_NULL, 0);
    crc = crc32(crc, out.data() + at, uInt(4 + n));
    put_be32(out, uint32_t(crc));
}

int paeth(int a, int b, int c) {
    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    if (pa <= pb && pa <= pc) return a;
    return pb <= pc ? b : c;
}

// Reverses the per-scanline filters of one (sub)image in place: rows of
// `rowbytes` bytes, each preceded by its filter type byte.
bool unfilter(uint8_t* data, size_t rows, size_t rowbytes, int bpp) {
    std::vector<uint8_t> zero(rowbytes, 0);
    const uint8_t* prev = zero.data();
    for (size_t r = 0; r < rows; ++r) {
        uint8_t* line = data + r * (rowbytes + 1);
        const int ft = line[0];
        uint8_t* x = line + 1;
        switch (ft) {
            case 0: break;
            case 1:
                for (size_t i = size_t(bpp); i < rowbytes; ++i) x[i] = uint8_t(x[i] + x[i - bpp]);
                break;
            case 2:
                for (size_t i = 0; i < rowbytes; ++i) x[i] = uint8_t(x[i] + prev[i]);
                break;
            case 3:
                for (size_t i = 0; i < rowbytes; ++i) {
                    const int a = i >= size_t(bpp) ? x[i - bpp] : 0;
                    x[i] = uint8_t(x[i] + ((a + prev[i]) >> 1));
                }
                break;
            case 4:
                for (size_t i = 0; i < rowbytes; ++i) {
                    const int a = i >= size_t(bpp) ? x[i - bpp] : 0, c = i >= size_t(bpp) ? prev[i - bpp] : 0;
                    x[i] = uint8_t(x[i] + paeth(a, prev[i], c));
                }
                break;
            default: return false;
        }
        prev = x;
    }
    return true;
}

// Sample s (0-based) of an unfiltered row at bit depth < 8 or == 8.
inline int sample(const uint8_t* row, size_t s, int depth) {
    if (depth == 8) return row[s];
    const size_t bit = s * size_t(depth);
    return (row[bit >> 3] >> (8 - depth - int(bit & 7))) & ((1 << depth) - 1);
}

}  // namespace

void write_pfm(const std::string& path, const GridF& image) {
    const int C = image.channels();
    if (C != 1 && C != 3) throw std::invalid_argument("write_pfm: only 1 or 3 channels supported");
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(path, "cannot open for writing");
    out << (C == 3 ? "PF" : "Pf") << "\n" << image.width() << " " << image.height() << "\n" << "-1.0\n";
    std::vector<float> row(size_t(image.width()) * C);
    for (int y = image.height() - 1; y >= 0; --y) {  // bottom-up on disk
        const Scalar* src = image.row(y);
        for (size_t i = 0; i < row.size(); ++i) row[i] = float(src[i]);
        if (!host_little_endian())
            for (auto& v : row) {
                uint32_t b;
                std::memcpy(&b, &v, 4);
                b = __builtin_bswap32(b);
                std::memcpy(&v, &b, 4);
            }
        out.write(reinterpret_cast<const char*>(row.data()), std::streamsize(row.size() * sizeof(float)));
    }
    if (!out) fail(path, "write failed");
}

GridF read_pfm(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(path, "cannot open");
    std::string magic;
    in >> magic;
    int channels = 0;
    if (magic == "PF")
        channels = 3;
    else if (magic == "Pf")
        channels = 1;
    else
        fail(path, "bad PFM magic at byte offset 0 (expected 'PF' or 'Pf')");
    int w = 0, h = 0;
    double scale = 0;
    in >> w >> h >> scale;
    if (!in || w <= 0 || h <= 0 || scale == 0) fail(path, "malformed PFM header");
    in.get();  // the single whitespace after the scale
    const bool swap = (scale < 0) != host_little_endian();
    GridF image(w, h, channels);
    std::vector<float> row(size_t(w) * channels);
    for (int y = h - 1; y >= 0; --y) {
        in.read(reinterpret_cast<char*>(row.data()), std::streamsize(row.size() * sizeof(float)));
        if (!in) fail(path, "truncated PFM payload at byte offset " + std::to_string(size_t(in.tellg())));
        Scalar* dst = image.row(y);
        for (size_t i = 0; i < row.size(); ++i) {
            float v = row[i];
            if (swap) {
                uint32_t b;
                std::memcpy(&b, &v, 4);
                b = __builtin_bswap32(b);
                std::memcpy(&v, &b, 4);
            }
            dst[i] = v;
        }
    }
    return image;
}

void write_png(const std::string& path, const GridU8& image) {
    const int C = image.channels();
    if (C != 1 && C != 3) throw std::invalid_argument("write_png: only 1 or 3 channels supported");
    std::FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) fail(path, "cannot open for writing");
    const size_t W = size_t(image.width()), H = size_t(image.height()), rb = W * size_t(C);
    std::vector<uint8_t> raw((rb + 1) * H);
    for (size_t y = 0; y < H; ++y) {  // filter type 0 (None) on every row
        raw[y * (rb + 1)] = 0;
        if (rb) std::memcpy(&raw[y * (rb + 1) + 1], image.row(int(y)), rb);
    }
    uLongf zn = compressBound(uLong(raw.size()));
    std::vector<uint8_t> z(zn);
    if (compress2(z.data(), &zn, raw.data(), uLong(raw.size()), Z_DEFAULT_COMPRESSION) != Z_OK) {
        std::fclose(fp);
        fail(path, "libpng write error");
    }
    std::vector<uint8_t> out(kPngSig, kPngSig + 8);
    uint8_t ihdr[13];
    const uint32_t w32 = uint32_t(W), h32 = uint32_t(H);
    for (int i = 0; i < 4; ++i) {
        ihdr[i] = uint8_t(w32 >> (24 - 8 * i));
        ihdr[4 + i] = uint8_t(h32 >> (24 - 8 * i));
    }
    ihdr[8] = 8;                  // bit depth
    ihdr[9] = C == 3 ? 2 : 0;     // RGB / gray
    ihdr[10] = ihdr[11] = ihdr[12] = 0;  // deflate, adaptive filtering, no interlace
    put_chunk(out, "IHDR", ihdr, 13);
    put_chunk(out, "IDAT", z.data(), zn);
    put_chunk(out, "IEND", nullptr, 0);
    const bool ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
    std::fclose(fp);
    if (!ok) fail(path, "libpng write error");
}

GridU8 read_png(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(path, "cannot open");
    std::vector<uint8_t> f((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (f.size() < 8 || std::memcmp(f.data(), kPngSig, 8) != 0) fail(path, "bad PNG signature at byte offset 0");
    const std::string rd = "libpng read error";

    // Chunks: IHDR first, PLTE / tRNS before the IDAT run, IEND last.  CRCs of
    // critical chunks are checked (libpng errors on them); ancillary ones are
    // skipped unchecked, as libpng discards them.
    uint32_t W = 0, H = 0;
    int depth = 0, ctype = -1, interlace = 0;
    std::vector<uint8_t> palette, idat;
    bool have_trns = false, have_ihdr = false, have_iend = false;
    size_t pos = 8;
    while (pos + 12 <= f.size()) {
        const uint32_t n = be32(&f[pos]);
        if (n > 0x7fffffffu || pos + 12 + size_t(n) > f.size()) fail(path, rd);
        const uint8_t* type = &f[pos + 4];
        const uint8_t* data = &f[pos + 8];
        const bool critical = (type[0] & 0x20) == 0;
        if (critical) {
            uLong crc = crc32(0L, Z_NULL, 0);
            crc = crc32(crc, type, uInt(4 + n));
            if (uint32_t(crc) != be32(data + n)) fail(path, rd);
        }
        const std::string t(reinterpret_cast<const char*>(type), 4);
        if (!have_ihdr && t != "IHDR") fail(path, rd);
        if (t == "IHDR") {
            if (have_ihdr || n != 13) fail(path, rd);
            have_ihdr = true;
            W = be32(data);
            H = be32(data + 4);
            depth = data[8];
            ctype = data[9];
            interlace = data[12];
            const bool ok_combo = (ctype == 0 && (depth == 1 || depth == 2 || depth == 4 || depth == 8 || depth == 16)) ||
                                  (ctype == 3 && (depth == 1 || depth == 2 || depth == 4 || depth == 8)) ||
                                  ((ctype == 2 || ctype == 4 || ctype == 6) && (depth == 8 || depth == 16));
            if (W == 0 || H == 0 || W > 0x7fffffffu || H > 0x7fffffffu || !ok_combo || data[10] != 0 || data[11] != 0 ||
                interlace > 1)
                fail(path, rd);
            // io_image.cpp:142-145: rejected before any pixel is decoded.
            if (depth == 16) fail(path, "16-bit PNG not supported");
        } else if (t == "PLTE") {
            if (n % 3 != 0 || n == 0 || n > 768) fail(path, rd);
            palette.assign(data, data + n);
        } else if (t == "tRNS") {
            have_trns = n > 0;
        } else if (t == "IDAT") {
            idat.insert(idat.end(), data, data + n);
        } else if (t == "IEND") {
            have_iend = true;
            break;
        } else if (critical) {
            fail(path, rd);  // unknown critical chunk
        }
        pos += 12 + size_t(n);
    }
    if (!have_ihdr || !have_iend || idat.empty()) fail(path, rd);
    if (ctype == 3 && palette.empty()) fail(path, rd);

    // Output channels after the reference's transforms (io_image.cpp:146-158):
    // palette -> RGB (RGBA when a tRNS chunk is present: png_set_palette_to_rgb
    // expands it, and the original colour type carries no alpha bit, so it is
    // not stripped), gray 1/2/4 -> gray 8, alpha stripped from gray+alpha/RGBA.
    const int in_ch = ctype == 0 ? 1 : ctype == 2 ? 3 : ctype == 3 ? 1 : ctype == 4 ? 2 : 4;
    const int out_ch = ctype == 3 ? (have_trns ? 4 : 3) : (ctype == 0 || ctype == 4 ? 1 : 3);
    if (out_ch != 1 && out_ch != 3) fail(path, "unsupported channel count " + std::to_string(out_ch));

    // Inflate the whole IDAT stream.
    const int bits_pp = in_ch * depth;
    const int bpp = std::max(1, bits_pp / 8);
    auto rowbytes_of = [&](size_t w) { return (w * size_t(bits_pp) + 7) / 8; };
    size_t expect = 0;
    static const int ax0[7] = {0, 4, 0, 2, 0, 1, 0}, ay0[7] = {0, 0, 4, 0, 2, 0, 1};
    static const int adx[7] = {8, 8, 4, 4, 2, 2, 1}, ady[7] = {8, 8, 8, 4, 4, 2, 2};
    if (interlace == 0) {
        expect = (rowbytes_of(W) + 1) * H;
    } else {
        for (int p = 0; p < 7; ++p) {
            const size_t pw = W > uint32_t(ax0[p]) ? (W - ax0[p] + adx[p] - 1) / adx[p] : 0;
            const size_t ph = H > uint32_t(ay0[p]) ? (H - ay0[p] + ady[p] - 1) / ady[p] : 0;
            if (pw && ph) expect += (rowbytes_of(pw) + 1) * ph;
        }
    }
    std::vector<uint8_t> raw(expect);
    {
        z_stream zs{};
        if (inflateInit(&zs) != Z_OK) fail(path, rd);
        zs.next_in = idat.data();
        zs.avail_in = uInt(idat.size());
        zs.next_out = raw.data();
        zs.avail_out = uInt(raw.size());
        const int st = inflate(&zs, Z_FINISH);
        const size_t got = raw.size() - zs.avail_out;
        inflateEnd(&zs);
        if ((st != Z_STREAM_END && st != Z_BUF_ERROR && st != Z_OK) || got != raw.size()) fail(path, rd);
    }

    GridU8 image(int(W), int(H), out_ch);
    auto put_pixel = [&](const uint8_t* row, size_t sx, uint8_t* dst) {
        if (ctype == 3) {
            const int idx = sample(row, sx, depth);
            const size_t np = palette.size() / 3;
            for (int c = 0; c < 3; ++c) dst[c] = size_t(idx) < np ? palette[size_t(idx) * 3 + c] : 0;
            if (out_ch == 4) dst[3] = 255;
        } else if (ctype == 0) {
            const int v = sample(row, sx, depth);
            dst[0] = uint8_t(depth == 8 ? v : depth == 4 ? v * 17 : depth == 2 ? v * 85 : v * 255);
        } else {
            const uint8_t* px = row + sx * size_t(in_ch);
            for (int c = 0; c < out_ch; ++c) dst[c] = px[c];  // alpha (last) dropped
        }
    };
    if (interlace == 0) {
        const size_t rb = rowbytes_of(W);
        if (!unfilter(raw.data(), H, rb, bpp)) fail(path, rd);
        for (size_t y = 0; y < H; ++y) {
            const uint8_t* row = raw.data() + y * (rb + 1) + 1;
            uint8_t* dst = image.row(int(y));
            for (size_t x = 0; x < W; ++x) put_pixel(row, x, dst + x * size_t(out_ch));
        }
    } else {  // Adam7: seven reduced images, each filtered on its own
        size_t off = 0;
        for (int p = 0; p < 7; ++p) {
            const size_t pw = W > uint32_t(ax0[p]) ? (W - ax0[p] + adx[p] - 1) / adx[p] : 0;
            const size_t ph = H > uint32_t(ay0[p]) ? (H - ay0[p] + ady[p] - 1) / ady[p] : 0;
            if (!pw || !ph) continue;
            const size_t rb = rowbytes_of(pw);
            if (!unfilter(raw.data() + off, ph, rb, bpp)) fail(path, rd);
            for (size_t r = 0; r < ph; ++r) {
                const uint8_t* row = raw.data() + off + r * (rb + 1) + 1;
                uint8_t* dst = image.row(int(ay0[p] + r * ady[p]));
                for (size_t i = 0; i < pw; ++i) put_pixel(row, i, dst + (ax0[p] + i * adx[p]) * size_t(out_ch));
            }
            off += (rb + 1) * ph;
        }
    }
    return image;
}

GridU8 to_u8(const GridF& image) {
    GridU8 out(image.width(), image.height(), image.channels());
    for (size_t i = 0; i < image.size(); ++i) {
        const Scalar v = std::clamp(image.storage()[i], Scalar(0), Scalar(1));
        out.storage()[i] = uint8_t(std::lround(v * 255.0));
    }
    return out;
}

GridF to_unit(const GridU8& image) {
    GridF out(image.width(), image.height(), image.channels());
    for (size_t i = 0; i < image.size(); ++i) out.storage()[i] = Scalar(image.storage()[i]) / 255.0;
    return out;
}

}  // namespace msplat
