// Signal files at the edges of the path (SURVEY 8f "next"): binary PGM (P5,
// 8/16-bit) and SVOL volumes, byte-compatible with the reference's
// image_io.hpp:9-24 / image_io.cpp:43-159 (same header grammar, same rounding
// and clamping on save, same FormatError conditions). Host code.
#pragma once
#include <cctype>
#include <cmath>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "common.cuh"

namespace slb {

// whitespace / '#'-comment separated PNM token (image_io.cpp:13-30)
static bool pnm_token(std::istream& in, std::string& tok) {
    tok.clear();
    int c = in.get();
    for (;;) {
        if (c == EOF) break;
        if (c == '#') {
            while (c != EOF && c != '\n') c = in.get();
        } else if (std::isspace(c)) {
            c = in.get();
        } else {
            break;
        }
    }
    while (c != EOF && !std::isspace(c)) {
        tok.push_back(static_cast<char>(c));
        c = in.get();
    }
    return !tok.empty();
}

static size_t pnm_size(const std::string& tok, const char* what) {
    size_t v = 0;
    for (char c : tok) {
        if (c < '0' || c > '9') throw SlError(SL_ERR_FORMAT, std::string("PGM: bad ") + what);
        v = v * 10 + static_cast<size_t>(c - '0');
    }
    return v;
}

struct PgmHeader {
    size_t rows = 0, cols = 0;
    int maxval = 0;
};

// Reads the header; leaves `in` at the first pixel byte.
static PgmHeader pgm_header(std::istream& in, const std::string& path) {
    std::string tok;
    if (!pnm_token(in, tok) || tok != "P5") throw SlError(SL_ERR_FORMAT, "not a binary PGM (P5) file: " + path);
    PgmHeader h;
    if (!pnm_token(in, tok)) throw SlError(SL_ERR_FORMAT, "PGM truncated: " + path);
    h.cols = pnm_size(tok, "width");
    if (!pnm_token(in, tok)) throw SlError(SL_ERR_FORMAT, "PGM truncated: " + path);
    h.rows = pnm_size(tok, "height");
    if (!pnm_token(in, tok)) throw SlError(SL_ERR_FORMAT, "PGM truncated: " + path);
    const size_t mv = pnm_size(tok, "maxval");
    if (h.cols == 0 || h.rows == 0 || mv == 0 || mv > 65535)
        throw SlError(SL_ERR_FORMAT, "PGM: bad header values: " + path);
    h.maxval = static_cast<int>(mv);
    return h;
}

static PgmHeader pgm_load(const std::string& path, double* out, long long cap) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw SlError(SL_ERR_FORMAT, "cannot open PGM file: " + path);
    const PgmHeader h = pgm_header(in, path);
    if (!out) return h;
    if (cap < static_cast<long long>(h.rows * h.cols)) throw SlError(SL_ERR_INVALID, "PGM: output buffer too small");
    const size_t bpp = h.maxval > 255 ? 2 : 1;
    std::vector<unsigned char> row(h.cols * bpp);
    for (size_t i = 0; i < h.rows; ++i) {
        if (!in.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(row.size())))
            throw SlError(SL_ERR_FORMAT, "PGM pixel data truncated: " + path);
        double* o = out + i * h.cols;
        for (size_t j = 0; j < h.cols; ++j)
            o[j] = bpp == 1 ? static_cast<double>(row[j]) : static_cast<double>((row[2 * j] << 8) | row[2 * j + 1]);
    }
    return h;
}

static void pgm_save(const double* px, size_t rows, size_t cols, const std::string& path, int maxval) {
    if (maxval <= 0 || maxval > 65535) throw SlError(SL_ERR_FORMAT, "PGM: maxval out of range");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw SlError(SL_ERR_FORMAT, "cannot write PGM file: " + path);
    out << "P5\n" << cols << ' ' << rows << '\n' << maxval << '\n';
    const bool wide = maxval > 255;
    std::vector<unsigned char> row(cols * (wide ? 2 : 1));
    for (size_t i = 0; i < rows; ++i) {
        for (size_t j = 0; j < cols; ++j) {
            const double v = std::min(static_cast<double>(maxval), std::max(0.0, std::round(px[i * cols + j])));
            const unsigned u = static_cast<unsigned>(v);
            if (wide) {
                row[2 * j] = static_cast<unsigned char>(u >> 8);
                row[2 * j + 1] = static_cast<unsigned char>(u & 0xff);
            } else {
                row[j] = static_cast<unsigned char>(u);
            }
        }
        out.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size()));
    }
    if (!out) throw SlError(SL_ERR_FORMAT, "PGM write failed: " + path);
}

// SVOL: "SVOL", u16 version 1, 3 x u32 dims, f64 samples, all little-endian
static void svol_load(const std::string& path, double* out, long long cap, long long dims[3]) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw SlError(SL_ERR_FORMAT, "cannot open SVOL file: " + path);
    unsigned char hdr[18];
    if (!in.read(reinterpret_cast<char*>(hdr), 4) || std::memcmp(hdr, "SVOL", 4) != 0)
        throw SlError(SL_ERR_FORMAT, "not an SVOL file: " + path);
    if (!in.read(reinterpret_cast<char*>(hdr + 4), 2)) throw SlError(SL_ERR_FORMAT, "SVOL truncated: " + path);
    if ((hdr[4] | (hdr[5] << 8)) != 1) throw SlError(SL_ERR_FORMAT, "SVOL: unsupported version: " + path);
    for (int a = 0; a < 3; ++a) {
        unsigned char b[4];
        if (!in.read(reinterpret_cast<char*>(b), 4)) throw SlError(SL_ERR_FORMAT, "SVOL truncated: " + path);
        dims[a] = static_cast<long long>(static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
                                         (static_cast<uint32_t>(b[2]) << 16) | (static_cast<uint32_t>(b[3]) << 24));
    }
    if (dims[0] == 0 || dims[1] == 0 || dims[2] == 0) throw SlError(SL_ERR_FORMAT, "SVOL: zero dims: " + path);
    if (!out) return;
    const long long n = dims[0] * dims[1] * dims[2];
    if (cap < n) throw SlError(SL_ERR_INVALID, "SVOL: output buffer too small");
    std::vector<unsigned char> buf(static_cast<size_t>(n) * 8);
    if (!in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size())))
        throw SlError(SL_ERR_FORMAT, "SVOL truncated: " + path);
    for (long long i = 0; i < n; ++i) {
        uint64_t u = 0;
        for (int k = 0; k < 8; ++k) u |= static_cast<uint64_t>(buf[static_cast<size_t>(i) * 8 + k]) << (8 * k);
        std::memcpy(out + i, &u, 8);
    }
}

static void svol_save(const double* v, const long long dims[3], const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw SlError(SL_ERR_FORMAT, "cannot write SVOL file: " + path);
    std::vector<unsigned char> buf;
    const long long n = dims[0] * dims[1] * dims[2];
    buf.reserve(18 + static_cast<size_t>(n) * 8);
    auto put = [&buf](uint64_t u, int bytes) {
        for (int k = 0; k < bytes; ++k) buf.push_back(static_cast<unsigned char>(u >> (8 * k)));
    };
    buf.insert(buf.end(), {'S', 'V', 'O', 'L'});
    put(1, 2);
    for (int a = 0; a < 3; ++a) put(static_cast<uint32_t>(dims[a]), 4);
    for (long long i = 0; i < n; ++i) {
        uint64_t u;
        std::memcpy(&u, v + i, 8);
        put(u, 8);
    }
    out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
    if (!out) throw SlError(SL_ERR_FORMAT, "SVOL write failed: " + path);
}

}  // namespace slb
