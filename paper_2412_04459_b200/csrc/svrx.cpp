// svrx.cpp — the SVRX checkpoint container (io.cpp:229-359) for device scenes.
//
// Layout, little-endian, exactly as save_checkpoint writes it (io.cpp:250-279):
//   "SVRX" | u32 version (1) | u32 header length | header JSON |
//   u64 code[N] | u8 level[N] | u32 corner_index[N][8] | f32 density[P] |
//   f32 sh[N][3(d+1)^2] | u32 crc32 (zlib) of everything before it.
// The header is nlohmann::ordered_json's dump() of {voxel_count, pool_count,
// sh_degree, bounds_center[3], bounds_size}; numbers are written the way its
// serializer does (integers plainly, doubles as the shortest round-trip
// digits with ".0" for integral values, exponent form outside [1e-4, 1e15)).
// The reader repeats load_checkpoint's checks in its order and with its
// messages (io.cpp:281-359), including the structural corner-key check.
#include <zlib.h>

#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "svrx.h"

namespace svrb {

namespace {

constexpr uint32_t kVersion = 1;

template <typename T>
void append(std::vector<uint8_t>& b, const T* p, size_t n) {
    const auto* c = reinterpret_cast<const uint8_t*>(p);
    b.insert(b.end(), c, c + n * sizeof(T));
}

template <typename T>
void take(const std::vector<uint8_t>& b, size_t& off, T* p, size_t n) {
    const size_t bytes = n * sizeof(T);
    if (off + bytes > b.size()) throw SvrxError("truncated checkpoint");
    std::memcpy(p, b.data() + off, bytes);
    off += bytes;
}

// nlohmann::json's float serialisation (shortest round-trip digits).
std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char digits[32];
    int exp10 = 0;
    for (int prec = 1; prec <= 17; ++prec) {
        char buf[48];
        std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
        if (std::strtod(buf, nullptr) == v || prec == 17) {
            // buf = [-]d.ddddde[+-]XX
            const char* p = buf;
            std::string d;
            for (; *p && *p != 'e'; ++p)
                if (*p >= '0' && *p <= '9') d.push_back(*p);
            exp10 = std::atoi(p + 1);
            while (d.size() > 1 && d.back() == '0') d.pop_back();
            std::snprintf(digits, sizeof digits, "%s", d.c_str());
            break;
        }
    }
    const std::string d = digits;
    const int k = int(d.size()), n = exp10 + 1;  // value = 0.d * 10^n
    std::string out = v < 0 ? "-" : "";
    if (k <= n && n <= 15) {  // integral: digits, zeros, ".0"
        out += d + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += d.substr(0, size_t(n)) + "." + d.substr(size_t(n));
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(size_t(-n), '0') + d;
    } else {
        out += d.substr(0, 1);
        if (k > 1) out += "." + d.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return out;
}

// Minimal JSON reader for the header's shape: an object of numbers and one
// array of numbers.
struct JsonValue {
    bool is_array = false;
    std::string num;  // the literal
    std::vector<std::string> items;
};

struct JsonReader {
    const char* p;
    const char* end;
    void ws() {
        while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
    }
    void expect(char c) {
        ws();
        if (p >= end || *p != c) throw SvrxError(std::string("expected '") + c + "'");
        ++p;
    }
    std::string str() {
        expect('"');
        std::string s;
        while (p < end && *p != '"') s.push_back(*p++);
        if (p >= end) throw SvrxError("unterminated string");
        ++p;
        return s;
    }
    std::string number() {
        ws();
        const char* b = p;
        while (p < end && (std::strchr("+-.eE", *p) || (*p >= '0' && *p <= '9'))) ++p;
        if (p == b) throw SvrxError("expected a number");
        return std::string(b, p);
    }
    std::map<std::string, JsonValue> object() {
        std::map<std::string, JsonValue> m;
        expect('{');
        ws();
        if (p < end && *p == '}') {
            ++p;
            return m;
        }
        for (;;) {
            const std::string k = str();
            expect(':');
            ws();
            JsonValue v;
            if (p < end && *p == '[') {
                ++p;
                v.is_array = true;
                ws();
                if (p < end && *p == ']') {
                    ++p;
                } else {
                    for (;;) {
                        v.items.push_back(number());
                        ws();
                        if (p < end && *p == ',') {
                            ++p;
                            continue;
                        }
                        expect(']');
                        break;
                    }
                }
            } else {
                v.num = number();
            }
            m[k] = v;
            ws();
            if (p < end && *p == ',') {
                ++p;
                continue;
            }
            expect('}');
            break;
        }
        ws();
        if (p != end) throw SvrxError("trailing characters");
        return m;
    }
};

const JsonValue& at(const std::map<std::string, JsonValue>& m, const char* k) {
    auto it = m.find(k);
    if (it == m.end()) throw SvrxError(std::string("missing key ") + k);
    return it->second;
}

}  // namespace

std::string svrx_header(uint64_t n, uint64_t p, int sh_degree, const double* bc, double bs) {
    return "{\"voxel_count\":" + std::to_string(n) + ",\"pool_count\":" + std::to_string(p) +
           ",\"sh_degree\":" + std::to_string(sh_degree) + ",\"bounds_center\":[" +
           json_double(bc[0]) + "," + json_double(bc[1]) + "," + json_double(bc[2]) +
           "],\"bounds_size\":" + json_double(bs) + "}";
}

std::vector<uint8_t> svrx_encode(const SvrxScene& s) {
    const std::string h = svrx_header(s.codes.size(), s.density.size(), s.sh_degree,
                                      s.bounds_center, s.bounds_size);
    std::vector<uint8_t> b;
    b.reserve(16 + h.size() + s.codes.size() * 41 + s.density.size() * 4 + s.sh.size() * 4);
    append(b, "SVRX", 4);
    const uint32_t version = kVersion, hlen = uint32_t(h.size());
    append(b, &version, 1);
    append(b, &hlen, 1);
    append(b, h.data(), h.size());
    append(b, s.codes.data(), s.codes.size());
    append(b, s.levels.data(), s.levels.size());
    append(b, s.corner_index.data(), s.corner_index.size());
    append(b, s.density.data(), s.density.size());
    append(b, s.sh.data(), s.sh.size());
    const uint32_t crc = uint32_t(crc32(0, b.data(), uInt(b.size())));
    append(b, &crc, 1);
    return b;
}

void svrx_write(const std::string& path, const std::vector<uint8_t>& b) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw SvrxError("cannot write " + path);
    out.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size()));
    if (!out) throw SvrxError("write failed for " + path);
}

SvrxScene svrx_read(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw SvrxError("cannot open " + path);
    std::vector<uint8_t> b((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (b.size() < 16) throw SvrxError("truncated checkpoint " + path);
    if (std::memcmp(b.data(), "SVRX", 4) != 0)
        throw SvrxError(path + ": not an SVRX checkpoint (bad magic)");
    uint32_t stored;
    std::memcpy(&stored, b.data() + b.size() - 4, 4);
    if (uint32_t(crc32(0, b.data(), uInt(b.size() - 4))) != stored)
        throw SvrxError(path + ": checksum failure");
    size_t off = 4;
    uint32_t version = 0, hlen = 0;
    take(b, off, &version, 1);
    take(b, off, &hlen, 1);
    if (version != kVersion)
        throw SvrxError(path + ": unsupported checkpoint version " + std::to_string(version));
    if (off + hlen > b.size()) throw SvrxError("truncated checkpoint " + path);
    std::map<std::string, JsonValue> h;
    SvrxScene s;
    size_t n = 0, p = 0;
    try {
        JsonReader r{reinterpret_cast<const char*>(b.data() + off),
                     reinterpret_cast<const char*>(b.data() + off + hlen)};
        h = r.object();
        n = size_t(std::stoull(at(h, "voxel_count").num));
        p = size_t(std::stoull(at(h, "pool_count").num));
        s.sh_degree = std::stoi(at(h, "sh_degree").num);
        const JsonValue& bc = at(h, "bounds_center");
        if (!bc.is_array || bc.items.size() != 3) throw SvrxError("bounds_center");
        for (int i = 0; i < 3; ++i) s.bounds_center[i] = std::strtod(bc.items[i].c_str(), nullptr);
        s.bounds_size = std::strtod(at(h, "bounds_size").num.c_str(), nullptr);
    } catch (const std::exception& e) {
        throw SvrxError(path + ": malformed checkpoint header: " + e.what());
    }
    off += hlen;
    if (s.sh_degree < 0 || s.sh_degree > 3) throw SvrxError(path + ": invalid sh_degree");
    const size_t stride = size_t(3 * (s.sh_degree + 1) * (s.sh_degree + 1));
    s.codes.resize(n);
    s.levels.resize(n);
    take(b, off, s.codes.data(), n);
    take(b, off, s.levels.data(), n);
    for (size_t i = 0; i < n; ++i) {  // to_voxel_index validates level and alignment
        const int lv = s.levels[i];
        if (lv < 1 || lv > 16) throw SvrxInvalid("octree level out of [1,16]");
        const int shift = 3 * (16 - lv);
        if (shift < 64 && (s.codes[i] & ((uint64_t(1) << shift) - 1)) != 0)
            throw SvrxInvalid("octpath has nonzero bits below its level");
        if ((s.codes[i] >> 48) != 0) throw SvrxInvalid("octpath code exceeds 48 bits");
    }
    s.corner_index.resize(n * 8);
    take(b, off, s.corner_index.data(), n * 8);
    s.density.resize(p);
    take(b, off, s.density.data(), p);
    s.sh.resize(n * stride);
    take(b, off, s.sh.data(), s.sh.size());
    if (off != b.size() - 4)
        throw SvrxError(path + ": checkpoint length disagrees with its header");
    return s;
}

// load_checkpoint's structural validation (io.cpp:342-357): every corner of
// every voxel maps to the pool entry its lattice key maps to elsewhere, and
// every pool entry is used. Levels were already checked by the caller.
void svrx_validate(const SvrxScene& s, const std::string& path) {
    const size_t n = s.codes.size(), p = s.density.size();
    std::vector<bool> used(p, false);
    std::unordered_map<uint64_t, uint32_t> seen;
    seen.reserve(n * 2);
    for (size_t vi = 0; vi < n; ++vi) {
        const int lv = s.levels[vi];
        uint64_t c = s.codes[vi] >> (3 * (16 - lv));
        uint32_t i = 0, j = 0, k = 0;
        for (int b = 0; b < lv; ++b) {  // to_voxel_index (octree.hpp:68-82)
            i |= uint32_t((c >> 2) & 1) << b;
            j |= uint32_t((c >> 1) & 1) << b;
            k |= uint32_t(c & 1) << b;
            c >>= 3;
        }
        const uint32_t step = uint32_t(1) << (16 - lv);  // corner_keys (octree.hpp:130-139)
        for (uint32_t cc = 0; cc < 8; ++cc) {
            const uint64_t key = (uint64_t((i + ((cc >> 2) & 1)) * step) << 34) |
                                 (uint64_t((j + ((cc >> 1) & 1)) * step) << 17) |
                                 uint64_t((k + (cc & 1)) * step);
            const uint32_t pi = s.corner_index[vi * 8 + cc];
            if (pi >= p) throw SvrxError(path + ": corner index out of range");
            used[pi] = true;
            auto [it, inserted] = seen.try_emplace(key, pi);
            if (!inserted && it->second != pi)
                throw SvrxError(path + ": inconsistent corner indexing");
        }
    }
    for (size_t q = 0; q < p; ++q)
        if (!used[q]) throw SvrxError(path + ": orphaned density pool entry");
}

}  // namespace svrb
