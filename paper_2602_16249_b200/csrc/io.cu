// AFT1 tensor files and checkpoints straight from / into device memory:
// write_aft / read_aft (proj/src/tensor_io.cpp:60-105; format include/affmae/tensor_io.hpp:11-13:
// "AFT1", u8 dtype 0 = b32 / 1 = b16emu / 2 = u8, u32 ndim, ndim x u64 extents, little-endian
// payload of f32 values or raw bytes) and save_checkpoint / load_checkpoint
// (proj/src/pipeline.cpp:757-797: one <name>.aft per parameter plus manifest.tsv lines
// "name<TAB>d0xd1..<TAB>precision<TAB>file").  Files written here are byte-identical to the
// reference's for the same values; the device side is one pinned staging copy per tensor.
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <sys/stat.h>

#include <cuda_fp16.h>

#include "common.cuh"

namespace affmae_b200 {

namespace {

bool put(FILE* f, const void* p, size_t n) { return std::fwrite(p, 1, n, f) == n; }
void le32(unsigned char* b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b[i] = (unsigned char)(v >> (8 * i));
}
void le64(unsigned char* b, uint64_t v) {
    for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
}
uint32_t rd32(const unsigned char* b) {
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}
uint64_t rd64(const unsigned char* b) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(b[i]) << (8 * i);
    return v;
}

// product of the extents, false on a negative extent or int64 overflow (payload bytes
// up to 4 * numel must fit too)
bool checked_numel(const int64_t* dims, int nd, int64_t* out) {
    int64_t n = 1;
    for (int i = 0; i < nd; ++i) {
        if (dims[i] < 0) return false;
        if (dims[i] && n > (INT64_MAX / 4) / dims[i]) return false;
        n *= dims[i];
    }
    *out = n;
    return true;
}

// create_directories (the reference's save_checkpoint, proj/src/pipeline.cpp:759)
bool make_dirs(const std::string& path) {
    std::string cur;
    size_t pos = 0;
    while (pos <= path.size()) {
        size_t nx = path.find('/', pos);
        if (nx == std::string::npos) nx = path.size();
        cur = path.substr(0, nx);
        if (!cur.empty() && ::mkdir(cur.c_str(), 0755) != 0 && errno != EEXIST) return false;
        pos = nx + 1;
    }
    struct stat st;
    return ::stat(path.c_str(), &st) == 0 && S_ISDIR(st.st_mode);
}

struct File {
    FILE* f;
    explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

int write_file(const char* path, int dtype, const int64_t* dims, int ndim, const void* payload, size_t bytes) {
    File out(path, "wb");
    if (!out.f) return fail(AFFMAE_ECONFIG, std::string("cannot open for write: ") + path);
    unsigned char hdr[4 + 1 + 4 + 8 * 8];
    std::memcpy(hdr, "AFT1", 4);
    hdr[4] = (unsigned char)dtype;
    le32(hdr + 5, uint32_t(ndim));
    for (int i = 0; i < ndim; ++i) le64(hdr + 9 + 8 * i, uint64_t(dims[i]));
    if (!put(out.f, hdr, size_t(9 + 8 * ndim)) || !put(out.f, payload, bytes))
        return fail(AFFMAE_ECONFIG, std::string("short write: ") + path);
    return AFFMAE_OK;
}

}  // namespace

// device fp32 values -> AFT1 (dtype 0 b32 or 1 b16emu: the payload is f32 either way), or
// device bytes -> AFT1 dtype 2
int aft_write(const char* path, const void* dev_src, const int64_t* dims, int ndim, int dtype, void* stream) {
    if (!path || !dims || (ndim > 0 && !dev_src)) return fail(AFFMAE_ECONFIG, "aft_write: null pointer");
    if (ndim < 0 || ndim > 8) return fail(AFFMAE_ECONFIG, "aft_write: ndim must be in [0, 8]");
    if (dtype < 0 || dtype > 2) return fail(AFFMAE_ECONFIG, "aft_write: dtype must be 0, 1 or 2");
    int64_t numel = 0;
    if (!checked_numel(dims, ndim, &numel)) return fail(AFFMAE_ECONFIG, "aft_write: bad extents");
    const size_t bytes = size_t(numel) * (dtype == 2 ? 1 : 4);
    std::vector<unsigned char> host(bytes);
    if (bytes && (cudaMemcpyAsync(host.data(), dev_src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)) !=
                      cudaSuccess ||
                  cudaStreamSynchronize(as_stream(stream)) != cudaSuccess))
        return fail(AFFMAE_ECUDA, "aft_write: D2H failed");
    // b16emu tensors hold binary16-representable values (round_b16, proj/src/tensor.cpp:167-172):
    // round the fp32 payload to nearest-even binary16 so the file matches the reference's
    if (dtype == 1) {
        float* f = reinterpret_cast<float*>(host.data());
        for (int64_t i = 0; i < numel; ++i)
            if (f[i] == f[i]) f[i] = __half2float(__float2half_rn(f[i]));  // NaN passes through (round_b16_scalar)
    }
    // the payload is little-endian f32 / bytes, which is the device layout (x86-64 / aarch64 hosts)
    return write_file(path, dtype, dims, ndim, host.data(), bytes);
}

int aft_read_header(const char* path, int* dtype, int* ndim, int64_t* dims) {
    if (!path || !dtype || !ndim || !dims) return fail(AFFMAE_ECONFIG, "aft_read_header: null pointer");
    File in(path, "rb");
    if (!in.f) return fail(AFFMAE_ECONFIG, std::string("cannot open: ") + path);
    unsigned char b[9];
    if (std::fread(b, 1, 9, in.f) != 9 || std::memcmp(b, "AFT1", 4) != 0)
        return fail(AFFMAE_ECONFIG, std::string("not an AFT1 file: ") + path);
    if (b[4] > 2) return fail(AFFMAE_ECONFIG, std::string("bad AFT1 dtype in ") + path);
    const uint32_t nd = rd32(b + 5);
    if (nd > 8) return fail(AFFMAE_ECONFIG, std::string("implausible AFT1 ndim in ") + path);
    unsigned char e[64];
    if (std::fread(e, 1, 8 * nd, in.f) != 8 * nd) return fail(AFFMAE_ECONFIG, std::string("truncated AFT1 file: ") + path);
    for (uint32_t i = 0; i < nd; ++i) {
        const uint64_t x = rd64(e + 8 * i);
        if (x > uint64_t(INT64_MAX)) return fail(AFFMAE_ECONFIG, std::string("implausible AFT1 extent in ") + path);
        dims[i] = int64_t(x);
    }
    *dtype = b[4];
    *ndim = int(nd);
    return AFFMAE_OK;
}

// AFT1 -> device fp32 [numel] (u8 payloads load as their byte values, as read_aft)
int aft_read(const char* path, float* dev_dst, int64_t capacity, int64_t* numel_out, void* stream) {
    int dtype = 0, nd = 0;
    int64_t dims[8];
    int rc = aft_read_header(path, &dtype, &nd, dims);
    if (rc) return rc;
    int64_t numel = 0;
    if (!checked_numel(dims, nd, &numel)) return fail(AFFMAE_ECONFIG, std::string("implausible AFT1 extents in ") + path);
    if (numel > capacity) return fail(AFFMAE_ECONFIG, std::string("aft_read: destination too small for ") + path);
    if (numel > 0 && !dev_dst) return fail(AFFMAE_ECONFIG, "aft_read: null destination");
    File in(path, "rb");
    if (!in.f || std::fseek(in.f, 0, SEEK_END) != 0) return fail(AFFMAE_ECONFIG, std::string("cannot open: ") + path);
    const long fsize = std::ftell(in.f);
    const int64_t payload = numel * (dtype == 2 ? 1 : 4);
    if (fsize < 0 || int64_t(fsize) - int64_t(9 + 8 * nd) < payload)
        return fail(AFFMAE_ECONFIG, std::string("truncated AFT1 file: ") + path);
    if (std::fseek(in.f, long(9 + 8 * nd), SEEK_SET) != 0) return fail(AFFMAE_ECONFIG, std::string("cannot seek: ") + path);
    std::vector<float> host(static_cast<size_t>(numel));
    if (dtype == 2) {
        std::vector<unsigned char> raw(static_cast<size_t>(numel));
        if (std::fread(raw.data(), 1, raw.size(), in.f) != raw.size())
            return fail(AFFMAE_ECONFIG, std::string("truncated AFT1 file: ") + path);
        for (size_t i = 0; i < raw.size(); ++i) host[i] = float(raw[i]);
    } else {
        std::vector<unsigned char> raw(static_cast<size_t>(numel) * 4);
        if (std::fread(raw.data(), 1, raw.size(), in.f) != raw.size())
            return fail(AFFMAE_ECONFIG, std::string("truncated AFT1 file: ") + path);
        for (size_t i = 0; i < size_t(numel); ++i) {
            const uint32_t v = rd32(raw.data() + 4 * i);
            std::memcpy(&host[i], &v, 4);
        }
    }
    if (numel && (cudaMemcpyAsync(dev_dst, host.data(), size_t(numel) * 4, cudaMemcpyHostToDevice,
                                  as_stream(stream)) != cudaSuccess ||
                  cudaStreamSynchronize(as_stream(stream)) != cudaSuccess))
        return fail(AFFMAE_ECUDA, "aft_read: H2D failed");
    if (numel_out) *numel_out = numel;
    return AFFMAE_OK;
}

// save_checkpoint (proj/src/pipeline.cpp:757-770) from device fp32 parameter buffers
int checkpoint_save(const char* dir, int n, const char* const* names, const float* const* dev_vals,
                    const int64_t* const* dims, const int* ndims, const int* precs, void* stream) {
    if (!dir || (n > 0 && (!names || !dev_vals || !dims || !ndims || !precs)))
        return fail(AFFMAE_ECONFIG, "checkpoint_save: null pointer");
    if (!make_dirs(dir)) return fail(AFFMAE_ECONFIG, std::string("cannot create checkpoint dir ") + dir);
    const std::string d(dir);
    std::string manifest;
    static const char* kPrec[3] = {"b32", "b16emu", "b64"};
    for (int i = 0; i < n; ++i) {
        if (precs[i] < 0 || precs[i] > 2) return fail(AFFMAE_ECONFIG, "checkpoint_save: bad precision");
        const std::string file = std::string(names[i]) + ".aft";
        // b64 tensors are stored as b32 (tensor_io.hpp:14); b16emu keeps its code
        int rc = aft_write((d + "/" + file).c_str(), dev_vals[i], dims[i], ndims[i], precs[i] == 1 ? 1 : 0, stream);
        if (rc) return rc;
        manifest += names[i];
        manifest += '\t';
        for (int k = 0; k < ndims[i]; ++k) manifest += (k ? "x" : "") + std::to_string(dims[i][k]);
        manifest += '\t';
        manifest += kPrec[precs[i]];
        manifest += '\t' + file + '\n';
    }
    File idx((d + "/manifest.tsv").c_str(), "wb");
    if (!idx.f || !put(idx.f, manifest.data(), manifest.size()))
        return fail(AFFMAE_ECONFIG, "cannot write checkpoint index in " + d);
    return AFFMAE_OK;
}

// load_checkpoint (proj/src/pipeline.cpp:772-797) into device fp32 parameter buffers:
// every manifest line must name one of `names` with the same element count, and every
// name must be present (the reference's ConfigError cases)
int checkpoint_load(const char* dir, int n, const char* const* names, float* const* dev_vals, const int64_t* numels,
                    void* stream) {
    if (!dir || (n > 0 && (!names || !dev_vals || !numels))) return fail(AFFMAE_ECONFIG, "checkpoint_load: null pointer");
    const std::string d(dir);
    File idx((d + "/manifest.tsv").c_str(), "rb");
    if (!idx.f) return fail(AFFMAE_ECONFIG, "no checkpoint index in " + d);
    std::string text;
    char buf[4096];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, idx.f)) > 0) text.append(buf, got);
    std::vector<char> seen(static_cast<size_t>(n), 0);
    size_t pos = 0;
    while (pos < text.size()) {
        size_t eol = text.find('\n', pos);
        if (eol == std::string::npos) eol = text.size();
        const std::string line = text.substr(pos, eol - pos);
        pos = eol + 1;
        if (line.empty()) continue;
        std::vector<std::string> f;
        size_t s = 0;
        for (int k = 0; k < 4; ++k) {
            const size_t t = line.find('\t', s);
            f.push_back(line.substr(s, t == std::string::npos ? std::string::npos : t - s));
            if (t == std::string::npos) break;
            s = t + 1;
        }
        if (f.size() < 4) return fail(AFFMAE_ECONFIG, "malformed checkpoint index line: " + line);
        int which = -1;
        for (int i = 0; i < n; ++i)
            if (f[0] == names[i]) which = i;
        if (which < 0) return fail(AFFMAE_ECONFIG, "checkpoint has unknown parameter: " + f[0]);
        // size check from the header BEFORE any payload reaches the live parameter
        int dt = 0, nd = 0;
        int64_t hd[8], numel = 0;
        int rc = aft_read_header((d + "/" + f[3]).c_str(), &dt, &nd, hd);
        if (rc) return rc;
        if (!checked_numel(hd, nd, &numel) || numel != numels[which])
            return fail(AFFMAE_ECONFIG, "checkpoint size mismatch for " + f[0]);
        rc = aft_read((d + "/" + f[3]).c_str(), dev_vals[which], numels[which], &numel, stream);
        if (rc) return rc;
        seen[size_t(which)] = 1;
    }
    for (int i = 0; i < n; ++i)
        if (!seen[size_t(i)]) return fail(AFFMAE_ECONFIG, std::string("checkpoint is missing parameter: ") + names[i]);
    return AFFMAE_OK;
}

}  // namespace affmae_b200
