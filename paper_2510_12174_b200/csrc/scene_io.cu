// Extended-PLY scene I/O (core/src/io_ply.cpp:122-263)
// straight to and from the packed device parameter layout.
//
// The header is parsed on the host exactly as io_ply.cpp:46-85 does (same
// accepted forms, same error texts).  The binary payload moves in one bulk
// read and one host->device copy; a decode kernel then transposes the AoS rows
// into the SoA segments of msplat_param_layout (any mix of double / float /
// (u)int8 / 16- / 32-bit columns, decoded as io_ply.cpp:87-111 does).  Saving
// is the reverse: an encode kernel writes the float64 rows of io_ply.cpp:122-162
// and the host writes them after the header.  Scene::validate's finiteness
// check runs on the device and names the first offending primitive.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

// Column type codes: 0 float64, 1 float32, 2 uint8, 3 int8, 4 uint16 (any
// 2-byte type, io_ply.cpp:104-108), 5 int32 (any 4-byte integer, :109-110).
struct ColMap {
    int32_t src_off;  // byte offset in the row, -1 = default value
    int32_t type;
    double def;
};

__device__ __forceinline__ double decode_col(const unsigned char* row, const ColMap& m) {
    if (m.src_off < 0) return m.def;
    const unsigned char* p = row + m.src_off;
    switch (m.type) {
        case 0: {
            double v;
            memcpy(&v, p, 8);
            return v;
        }
        case 1: {
            float v;
            memcpy(&v, p, 4);
            return double(v);
        }
        case 2:
            return double(*p);
        case 3:
            return double(*reinterpret_cast<const signed char*>(p));
        case 4: {
            uint16_t v;
            memcpy(&v, p, 2);
            return double(v);
        }
        default: {
            int32_t v;
            memcpy(&v, p, 4);
            return double(v);
        }
    }
}

// packed[e] for every element e of the n x P packed layout: column maps are per
// packed column (P of them), i.e. per (segment, component).
template <typename Real>
__global__ void ply_decode_kernel(int64_t n, int P, const int64_t* __restrict__ seg_off, const int* __restrict__ seg_w,
                                  const ColMap* __restrict__ maps, const unsigned char* __restrict__ payload,
                                  int64_t row_size, Real* __restrict__ packed) {
    const int64_t total = n * P;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        // locate the segment of packed element e
        int s = 0;
        while (s < 6 && e >= seg_off[s + 1]) ++s;
        const int64_t r = e - seg_off[s];
        const int w = seg_w[s];
        const int64_t v = r / w;
        const int comp = int(r - v * w);
        int col = 0;
        for (int q = 0; q < s; ++q) col += seg_w[q];
        packed[e] = Real(decode_col(payload + v * row_size, maps[col + comp]));
    }
}

// One float64 row per Gaussian in the io_ply.cpp:141-160 column order.
template <typename Real>
__global__ void ply_encode_kernel(int64_t n, int C, int K, const Real* __restrict__ packed, double* __restrict__ rows) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Real* means = packed;
    const Real* quats = means + 3 * n;
    const Real* logs = quats + 4 * n;
    const Real* opac = logs + 3 * n;
    const Real* kk = opac + n;
    const Real* sh = kk + n;
    const Real* sem = sh + size_t(3) * K * n;
    const int W = 3 + 3 + 3 * (K - 1) + 1 + 3 + 4 + C + 1;
    double* row = rows + i * W;
    int o = 0;
    for (int j = 0; j < 3; ++j) row[o++] = double(means[3 * i + j]);
    for (int c = 0; c < 3; ++c) row[o++] = double(sh[(i * 3 + c) * K]);
    for (int c = 0; c < 3; ++c)
        for (int j = 1; j < K; ++j) row[o++] = double(sh[(i * 3 + c) * K + j]);
    row[o++] = double(opac[i]);
    for (int j = 0; j < 3; ++j) row[o++] = double(logs[3 * i + j]);
    for (int j = 0; j < 4; ++j) row[o++] = double(quats[4 * i + j]);
    for (int c = 0; c < C; ++c) row[o++] = double(sem[i * C + c]);
    row[o++] = double(kk[i]);
}

// Smallest primitive index with a non-finite field (scene.cpp:22-40).
template <typename Real>
__global__ void first_nonfinite_kernel(int64_t n, int P, const int64_t* __restrict__ seg_off,
                                       const int* __restrict__ seg_w, const Real* __restrict__ packed,
                                       unsigned long long* first) {
    const int64_t total = n * P;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        if (isfinite(packed[e])) continue;
        int s = 0;
        while (s < 6 && e >= seg_off[s + 1]) ++s;
        const int64_t v = (e - seg_off[s]) / seg_w[s];
        atomicMin(first, (unsigned long long)v);
    }
}

struct Prop {
    std::string name, type;
    size_t size = 0;
};

size_t type_size(const std::string& t) {  // io_ply.cpp:34-44
    if (t == "float" || t == "float32" || t == "int" || t == "int32" || t == "uint" || t == "uint32") return 4;
    if (t == "double" || t == "float64") return 8;
    if (t == "char" || t == "int8" || t == "uchar" || t == "uint8") return 1;
    if (t == "short" || t == "int16" || t == "ushort" || t == "uint16") return 2;
    return 0;
}

int type_code(const Prop& p) {  // io_ply.cpp:87-111
    if (p.size == 8) return 0;
    if (p.type == "float" || p.type == "float32") return 1;
    if (p.type == "uchar" || p.type == "uint8") return 2;
    if (p.type == "char" || p.type == "int8") return 3;
    if (p.size == 2) return 4;
    return 5;
}

bool read_line(FILE* f, std::string& line) {
    line.clear();
    int c;
    bool any = false;
    while ((c = std::fgetc(f)) != EOF) {
        any = true;
        if (c == '\n') return true;
        line.push_back(char(c));
    }
    return any;
}

struct Header {
    size_t vertex_count = 0;
    std::vector<Prop> props;
    size_t row_size = 0;
};

// io_ply.cpp:46-85; returns "" or the error text (without the path prefix).
std::string read_header(FILE* f, Header& h) {
    std::string line;
    if (!read_line(f, line) || line != "ply") return "not a PLY file (missing 'ply' magic)";
    if (!read_line(f, line) || line != "format binary_little_endian 1.0")
        return "unsupported PLY format (need binary_little_endian 1.0)";
    bool in_vertex = false;
    while (read_line(f, line)) {
        std::istringstream ls(line);
        std::string word;
        ls >> word;
        if (word == "end_header") break;
        if (word == "comment") continue;
        if (word == "element") {
            std::string name;
            size_t count = 0;
            ls >> name >> count;
            in_vertex = name == "vertex";
            if (in_vertex)
                h.vertex_count = count;
            else if (count > 0)
                return "unsupported non-vertex element '" + name + "'";
        } else if (word == "property") {
            if (!in_vertex) continue;
            std::string type, name;
            ls >> type >> name;
            if (type == "list") return "list properties are not supported";
            const size_t size = type_size(type);
            if (size == 0) return "unknown property type '" + type + "'";
            h.props.push_back({name, type, size});
            h.row_size += size;
        }
    }
    if (h.props.empty()) return "no vertex properties found";
    return "";
}

struct SceneLayout {
    int C = 0, deg = 0, K = 1, rest = 0;
    bool has_k = false;
    std::map<std::string, int> index;
};

// io_ply.cpp:170-211: required columns, SH degree, class count.
std::string scene_layout(const Header& h, SceneLayout& L, const std::string& path, bool warn) {
    for (size_t i = 0; i < h.props.size(); ++i) L.index[h.props[i].name] = int(i);
    for (const char* r : {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
                          "rot_0", "rot_1", "rot_2", "rot_3"})
        if (!L.index.count(r)) return std::string("missing required property '") + r + "'";
    while (L.index.count("f_rest_" + std::to_string(L.rest))) ++L.rest;
    if (L.rest % 3 != 0) return "f_rest_* count " + std::to_string(L.rest) + " is not a multiple of 3";
    L.K = 1 + L.rest / 3;
    L.deg = int(std::lround(std::sqrt(double(L.K)))) - 1;
    if ((L.deg + 1) * (L.deg + 1) != L.K || L.deg > 3)
        return "f_rest_* count " + std::to_string(L.rest) + " does not match an SH degree in [0,3]";
    while (L.index.count("sem_" + std::to_string(L.C))) ++L.C;
    L.has_k = L.index.count("grad_k") > 0;
    const size_t known = 14 + size_t(L.rest) + size_t(L.C) + (L.has_k ? 1 : 0);
    if (warn && h.props.size() > known)
        for (const Prop& p : h.props) {
            const std::string& n = p.name;
            const bool recognized = n == "x" || n == "y" || n == "z" || n == "opacity" || n == "grad_k" ||
                                    n.rfind("f_dc_", 0) == 0 || n.rfind("f_rest_", 0) == 0 ||
                                    n.rfind("scale_", 0) == 0 || n.rfind("rot_", 0) == 0 || n.rfind("sem_", 0) == 0;
            if (!recognized)
                std::fprintf(stderr, "msplat: %s: ignoring unknown property '%s'\n", path.c_str(), n.c_str());
        }
    return "";
}

}  // namespace

IoResult ply_scene_info(const char* path, int64_t* n, int* C, int* deg) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return {2, std::string(path) + ": cannot open"};
    Header h;
    std::string err = read_header(f, h);
    std::fclose(f);
    if (!err.empty()) return {2, std::string(path) + ": " + err};
    SceneLayout L;
    if (!(err = scene_layout(h, L, path, false)).empty()) return {2, std::string(path) + ": " + err};
    *n = int64_t(h.vertex_count);
    *C = L.C;
    *deg = L.deg;
    return {};
}

template <typename Real>
IoResult ply_load_scene(const char* path, Real* packed, cudaStream_t s, DeviceError*) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return {2, std::string(path) + ": cannot open"};
    Header h;
    std::string err = read_header(f, h);
    SceneLayout L;
    if (err.empty()) err = scene_layout(h, L, path, true);
    if (!err.empty()) {
        std::fclose(f);
        return {2, std::string(path) + ": " + err};
    }
    const int64_t n = int64_t(h.vertex_count);
    std::vector<unsigned char> payload(size_t(n) * h.row_size);
    const size_t got = payload.empty() ? 0 : std::fread(payload.data(), 1, payload.size(), f);
    std::fclose(f);
    if (got < payload.size())
        return {2, std::string(path) + ": truncated payload at vertex " + std::to_string(got / h.row_size)};
    // per packed column: source column of the row (io_ply.cpp:228-246)
    std::vector<size_t> offs(h.props.size());
    for (size_t i = 0, o = 0; i < h.props.size(); o += h.props[i].size, ++i) offs[i] = o;
    auto col = [&](const std::string& name) {
        const int i = L.index.at(name);
        return ColMap{int32_t(offs[size_t(i)]), type_code(h.props[size_t(i)]), 0.0};
    };
    const int K = L.K, C = L.C, P = 12 + 3 * K + C;
    std::vector<ColMap> maps;
    for (const char* c : {"x", "y", "z"}) maps.push_back(col(c));
    for (int j = 0; j < 4; ++j) maps.push_back(col("rot_" + std::to_string(j)));
    for (int j = 0; j < 3; ++j) maps.push_back(col("scale_" + std::to_string(j)));
    maps.push_back(col("opacity"));
    maps.push_back(L.has_k ? col("grad_k") : ColMap{-1, 0, 0.9});
    for (int c = 0; c < 3; ++c)
        for (int j = 0; j < K; ++j)
            maps.push_back(j == 0 ? col("f_dc_" + std::to_string(c))
                                  : col("f_rest_" + std::to_string(c * (K - 1) + j - 1)));
    for (int c = 0; c < C; ++c) maps.push_back(col("sem_" + std::to_string(c)));
    const int seg_w[7] = {3, 4, 3, 1, 1, 3 * K, C};
    int64_t seg_off[8];
    seg_off[0] = 0;
    for (int i = 0; i < 7; ++i) seg_off[i + 1] = seg_off[i] + n * seg_w[i];
    if (n == 0) return {};
    void *d_payload = nullptr, *d_maps = nullptr, *d_off = nullptr, *d_w = nullptr, *d_first = nullptr;
    cudaMalloc(&d_payload, payload.size());
    cudaMalloc(&d_maps, maps.size() * sizeof(ColMap));
    cudaMalloc(&d_off, sizeof seg_off);
    cudaMalloc(&d_w, sizeof seg_w);
    cudaMalloc(&d_first, 8);
    cudaMemcpyAsync(d_payload, payload.data(), payload.size(), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_maps, maps.data(), maps.size() * sizeof(ColMap), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_off, seg_off, sizeof seg_off, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_w, seg_w, sizeof seg_w, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(d_first, 0xff, 8, s);
    const int64_t total = n * P;
    const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32));
    ply_decode_kernel<Real><<<blocks, 256, 0, s>>>(n, P, static_cast<int64_t*>(d_off), static_cast<int*>(d_w),
                                                   static_cast<ColMap*>(d_maps),
                                                   static_cast<unsigned char*>(d_payload), int64_t(h.row_size), packed);
    first_nonfinite_kernel<Real><<<blocks, 256, 0, s>>>(n, P, static_cast<int64_t*>(d_off), static_cast<int*>(d_w),
                                                        packed, static_cast<unsigned long long*>(d_first));
    count_launches(2);
    unsigned long long first = ~0ull;
    cudaMemcpyAsync(&first, d_first, 8, cudaMemcpyDeviceToHost, s);
    const cudaError_t ce = cudaStreamSynchronize(s);
    cudaFree(d_payload);
    cudaFree(d_maps);
    cudaFree(d_off);
    cudaFree(d_w);
    cudaFree(d_first);
    if (ce != cudaSuccess) return {4, std::string("CUDA error: ") + cudaGetErrorString(ce)};
    if (first != ~0ull)  // scene.validate() at the end of load_scene_ply (io_ply.cpp:262)
        return {1, "Scene: primitive " + std::to_string(first) + " has non-finite fields"};
    return {};
}

template <typename Real>
IoResult ply_save_scene(const char* path, int64_t n, int C, int deg, const Real* packed, cudaStream_t s) {
    const int K = (deg + 1) * (deg + 1), P = 12 + 3 * K + C;
    const int seg_w[7] = {3, 4, 3, 1, 1, 3 * K, C};
    int64_t seg_off[8];
    seg_off[0] = 0;
    for (int i = 0; i < 7; ++i) seg_off[i + 1] = seg_off[i] + n * seg_w[i];
    const int W = 3 + 3 + 3 * (K - 1) + 1 + 3 + 4 + C + 1;
    std::vector<double> rows(size_t(n) * W);
    if (n > 0) {  // scene.validate() first (io_ply.cpp:123)
        void *d_off = nullptr, *d_w = nullptr, *d_first = nullptr, *d_rows = nullptr;
        cudaMalloc(&d_off, sizeof seg_off);
        cudaMalloc(&d_w, sizeof seg_w);
        cudaMalloc(&d_first, 8);
        cudaMalloc(&d_rows, rows.size() * 8);
        cudaMemcpyAsync(d_off, seg_off, sizeof seg_off, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_w, seg_w, sizeof seg_w, cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(d_first, 0xff, 8, s);
        const int64_t total = n * P;
        const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32));
        first_nonfinite_kernel<Real><<<blocks, 256, 0, s>>>(n, P, static_cast<int64_t*>(d_off),
                                                            static_cast<int*>(d_w), packed,
                                                            static_cast<unsigned long long*>(d_first));
        ply_encode_kernel<Real><<<unsigned((n + 255) / 256), 256, 0, s>>>(n, C, K, packed,
                                                                          static_cast<double*>(d_rows));
        count_launches(2);
        unsigned long long first = ~0ull;
        cudaMemcpyAsync(&first, d_first, 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(rows.data(), d_rows, rows.size() * 8, cudaMemcpyDeviceToHost, s);
        const cudaError_t ce = cudaStreamSynchronize(s);
        cudaFree(d_off);
        cudaFree(d_w);
        cudaFree(d_first);
        cudaFree(d_rows);
        if (ce != cudaSuccess) return {4, std::string("CUDA error: ") + cudaGetErrorString(ce)};
        if (first != ~0ull) return {1, "Scene: primitive " + std::to_string(first) + " has non-finite fields"};
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) return {2, std::string(path) + ": cannot open for writing"};
    std::string hdr = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(n) + "\n";
    auto prop = [&](const std::string& name) { hdr += "property double " + name + "\n"; };
    for (const char* c : {"x", "y", "z"}) prop(c);
    for (int i = 0; i < 3; ++i) prop("f_dc_" + std::to_string(i));
    for (int i = 0; i < 3 * (K - 1); ++i) prop("f_rest_" + std::to_string(i));
    prop("opacity");
    for (int i = 0; i < 3; ++i) prop("scale_" + std::to_string(i));
    for (int i = 0; i < 4; ++i) prop("rot_" + std::to_string(i));
    for (int i = 0; i < C; ++i) prop("sem_" + std::to_string(i));
    prop("grad_k");
    hdr += "end_header\n";
    bool ok = std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
    if (ok && !rows.empty()) ok = std::fwrite(rows.data(), 8, rows.size(), f) == rows.size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return {2, std::string(path) + ": write failed"};
    return {};
}

template IoResult ply_load_scene<float>(const char*, float*, cudaStream_t, DeviceError*);
template IoResult ply_load_scene<double>(const char*, double*, cudaStream_t, DeviceError*);
template IoResult ply_save_scene<float>(const char*, int64_t, int, int, const float*, cudaStream_t);
template IoResult ply_save_scene<double>(const char*, int64_t, int, int, const double*, cudaStream_t);

}  // namespace msplat_cuda
