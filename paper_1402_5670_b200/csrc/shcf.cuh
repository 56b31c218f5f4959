// SHCF coefficient-file wire format (SURVEY 8f "next"; transform.cpp:127-269):
// magic "SHCF", u16 version 1, u8 dimensionality, u32 dims, u32 band count,
// per band (u8 kind, i32 scale, i32 k1/shear, i32 k2/0), then the bands as
// little-endian f64, row-major. Host-side, byte-identical to the reference.
#pragma once
#include <cstring>
#include <vector>

#include "common.cuh"

namespace slb {

static size_t shcf_bytes(const System& s, int nbands) {
    if (nbands < 0) throw SlError(SL_ERR_SHAPE, "serialize: negative band count");
    return 4 + 2 + 1 + 4 * static_cast<size_t>(s.ndim) + 4 + 13 * static_cast<size_t>(nbands) +
           8 * static_cast<size_t>(nbands) * static_cast<size_t>(s.nreal);
}
static size_t shcf_header_bytes(const System& s, int nbands);

template <class T>
static void put_le(unsigned char*& p, T v) {
    using U = std::make_unsigned_t<T>;
    U u;
    std::memcpy(&u, &v, sizeof(T));
    for (size_t i = 0; i < sizeof(T); ++i) *p++ = static_cast<unsigned char>(u >> (8 * i));
}

template <class T>
static T get_le(const unsigned char*& p, const unsigned char* end) {
    if (static_cast<size_t>(end - p) < sizeof(T)) throw SlError(SL_ERR_FORMAT, "coefficient stream truncated");
    using U = std::make_unsigned_t<T>;
    U u = 0;
    for (size_t i = 0; i < sizeof(T); ++i) u |= static_cast<U>(*p++) << (8 * i);
    T v;
    std::memcpy(&v, &u, sizeof(T));
    return v;
}

static size_t shcf_header_bytes(const System& s, int nbands) {
    return 4 + 2 + 1 + 4 * static_cast<size_t>(s.ndim) + 4 + 13 * static_cast<size_t>(nbands);
}

// header + index records of the handle's bands [lo, hi); returns the end
static unsigned char* shcf_write_header(const System& s, unsigned char* out) {
    unsigned char* p = out;
    std::memcpy(p, "SHCF", 4);
    p += 4;
    put_le<uint16_t>(p, 1);
    put_le<uint8_t>(p, static_cast<uint8_t>(s.ndim));
    for (int a = 0; a < s.ndim; ++a) put_le<uint32_t>(p, static_cast<uint32_t>(s.n[a]));
    put_le<uint32_t>(p, static_cast<uint32_t>(s.nb()));
    for (int i = s.lo; i < s.hi; ++i) {
        const Record& r = s.index[static_cast<size_t>(i)];
        put_le<uint8_t>(p, static_cast<uint8_t>(r.kind));
        put_le<int32_t>(p, r.scale);
        put_le<int32_t>(p, r.k1);
        put_le<int32_t>(p, s.ndim == 2 ? 0 : r.k2);
    }
    return p;
}

// f64 samples, little-endian
static void shcf_write_data(const double* v, size_t count, unsigned char* p) {
    for (size_t i = 0; i < count; ++i) {
        uint64_t u;
        std::memcpy(&u, v + i, 8);
        put_le<uint64_t>(p, u);
    }
}
static void shcf_read_data(const unsigned char* p, size_t count, double* v) {
    for (size_t i = 0; i < count; ++i) {
        uint64_t u = 0;
        for (int k = 0; k < 8; ++k) u |= static_cast<uint64_t>(p[8 * i + k]) << (8 * k);
        std::memcpy(v + i, &u, 8);
    }
}

// bands = the handle's shard [lo, hi) records (a full system writes all R)
static void shcf_serialize(const System& s, const double* coeffs, int nbands, unsigned char* out) {
    if (nbands != s.nb()) throw SlError(SL_ERR_SHAPE, "serialize: stack does not match the system");
    unsigned char* p = shcf_write_header(s, out);
    shcf_write_data(coeffs, static_cast<size_t>(nbands) * static_cast<size_t>(s.nreal), p);
}

static void shcf_deserialize(const System& s, const unsigned char* in, size_t len, double* coeffs, int nbands) {
    const unsigned char* p = in;
    const unsigned char* end = in + len;
    if (len < 4 || std::memcmp(p, "SHCF", 4) != 0) throw SlError(SL_ERR_FORMAT, "coefficient stream: bad magic");
    p += 4;
    if (get_le<uint16_t>(p, end) != 1) throw SlError(SL_ERR_FORMAT, "coefficient stream: unsupported version");
    const int dim = get_le<uint8_t>(p, end);
    if (dim != 2 && dim != 3) throw SlError(SL_ERR_FORMAT, "coefficient stream: bad dimensionality");
    if (dim != s.ndim) throw SlError(SL_ERR_FORMAT, "coefficient stream: dimensionality differs from the system");
    uint32_t dims[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) dims[a] = get_le<uint32_t>(p, end);
    const int count = static_cast<int>(get_le<uint32_t>(p, end));
    for (int a = 0; a < dim; ++a)
        if (dims[a] == 0 || count == 0) throw SlError(SL_ERR_FORMAT, "coefficient stream: empty dims or band count");
    for (int a = 0; a < dim; ++a)
        if (static_cast<int>(dims[a]) != s.n[a])
            throw SlError(SL_ERR_SHAPE, "coefficient stream: dims do not match the system");
    if (count != nbands || count != s.nb()) throw SlError(SL_ERR_SHAPE, "coefficient stream: band count mismatch");
    for (int i = 0; i < count; ++i) {
        const int kind = get_le<uint8_t>(p, end);
        const bool ok = dim == 2 ? kind <= 2 : (kind == 0 || (kind >= 3 && kind <= 5));
        if (!ok) throw SlError(SL_ERR_FORMAT, "coefficient stream: bad filter kind");
        const int scale = get_le<int32_t>(p, end), k1 = get_le<int32_t>(p, end), k2 = get_le<int32_t>(p, end);
        const Record& r = s.index[static_cast<size_t>(s.lo + i)];
        if (r.kind != kind || r.scale != scale || r.k1 != k1 || (dim == 3 && r.k2 != k2))
            throw SlError(SL_ERR_SHAPE, "coefficient stream: index records differ from the system");
    }
    if (!coeffs) return;  // header-only validation (streaming reader)
    const size_t nd = static_cast<size_t>(count) * static_cast<size_t>(s.nreal);
    if (static_cast<size_t>(end - p) < 8 * nd) throw SlError(SL_ERR_FORMAT, "coefficient stream truncated");
    shcf_read_data(p, nd, coeffs);
}

}  // namespace slb
