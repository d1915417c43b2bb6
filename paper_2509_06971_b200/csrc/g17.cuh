// g17.cuh -- exact "%.17g" formatting of an IEEE double, host and device.
//
// The reference writes every field value with snprintf("%.17g")
// (field_io.cpp:15-19): 17 significant digits, correctly rounded from the exact
// binary value (ties to even), %f style when the decimal exponent X satisfies
// -4 <= X < 17 and %e style otherwise (at least two exponent digits), trailing
// zeros and a bare '.' removed; "inf", "-inf", "nan", "-nan" for the
// non-finite values.  This header reproduces glibc's output byte for byte:
//
//   * D = round(|v| * 10^(16-X)) from the 192-bit product of the 53-bit
//     significand and a 128-bit power of ten (pow10_table.inc, floor-truncated,
//     exact for 10^0 .. 10^55): the fraction of the product decides the rounding
//     unless it lies within the table's truncation error of one half;
//   * those rare near-midpoint cases are settled exactly by comparing |v| with
//     the decimal midpoint in multi-precision integers (m 2^e against
//     (2D+1) 5^q 2^(q-1), q = X-16).
//
// Compiled for the device (the writers in writers.cuh) and for the host (the
// CPU test tests/cpp/test_g17.cpp checks it against snprintf).
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define G17_HD __host__ __device__ __forceinline__
#else
#define G17_HD inline
#endif

namespace petto_b200 {
namespace g17 {

struct Pow10Entry {
    unsigned long long hi, lo;
    int e;      // 10^k ~= (hi:lo) * 2^e
    int exact;  // (hi:lo) * 2^e == 10^k
};

#if defined(__CUDACC__)
#define G17_TABLE_QUAL __device__ __constant__ const
#include "pow10_table.inc"
#undef G17_TABLE_QUAL
#define G17_TABLE_QUAL static const
namespace host {
#include "pow10_table.inc"
}
#else
#define G17_TABLE_QUAL static const
namespace host {
#include "pow10_table.inc"
}
#endif

G17_HD const Pow10Entry& pow10(int k) {
#if defined(__CUDA_ARCH__)
    return kPow10[k - POW10_MIN];
#else
    return host::kPow10[k - POW10_MIN];
#endif
}

G17_HD unsigned long long mulhi64(unsigned long long a, unsigned long long b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return (unsigned long long)(((unsigned __int128)a * b) >> 64);
#endif
}

G17_HD int clz64(unsigned long long x) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

// ---------------------------------------------------------------- bignum
// Little-endian 32-bit limbs; big enough for 5^341 * 2^53 * 2^1200.
constexpr int BN_LIMBS = 80;
struct Big {
    uint32_t w[BN_LIMBS];
    int n;
};
G17_HD void big_set(Big& a, unsigned long long v) {
    a.w[0] = (uint32_t)v;
    a.w[1] = (uint32_t)(v >> 32);
    a.n = a.w[1] ? 2 : (a.w[0] ? 1 : 0);
}
G17_HD void big_mul_small(Big& a, uint32_t m) {
    unsigned long long carry = 0;
    for (int i = 0; i < a.n; ++i) {
        const unsigned long long p = (unsigned long long)a.w[i] * m + carry;
        a.w[i] = (uint32_t)p;
        carry = p >> 32;
    }
    if (carry) a.w[a.n++] = (uint32_t)carry;
}
G17_HD void big_mul_pow5(Big& a, int q) {
    while (q >= 13) {
        big_mul_small(a, 1220703125u);  // 5^13
        q -= 13;
    }
    uint32_t m = 1;
    while (q-- > 0) m *= 5;
    if (m != 1) big_mul_small(a, m);
}
G17_HD void big_shl(Big& a, int s) {
    if (a.n == 0 || s == 0) return;
    const int limbs = s >> 5, bits = s & 31;
    if (bits) {
        uint32_t carry = 0;
        for (int i = 0; i < a.n; ++i) {
            const uint32_t v = a.w[i];
            a.w[i] = (v << bits) | carry;
            carry = v >> (32 - bits);
        }
        if (carry) a.w[a.n++] = carry;
    }
    if (limbs) {
        for (int i = a.n - 1; i >= 0; --i) a.w[i + limbs] = a.w[i];
        for (int i = 0; i < limbs; ++i) a.w[i] = 0;
        a.n += limbs;
    }
}
G17_HD int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

// sign of m 2^e - (2d+1) 10^q / 2, exactly
G17_HD int cmp_midpoint(unsigned long long m, int e, unsigned long long d, int q) {
    Big a, b;
    big_set(a, m);
    big_set(b, 2 * d + 1);
    // a 2^e  vs  b 5^q 2^(q-1)
    if (q >= 0) big_mul_pow5(b, q);
    else big_mul_pow5(a, -q);
    const int s = e - (q - 1);  // a 2^s vs b
    if (s >= 0) big_shl(a, s);
    else big_shl(b, -s);
    return big_cmp(a, b);
}

// round(m 2^e 10^k) with m < 2^53 normalised (bit 52 set); bit 63 set: the
// fraction is within the table error of one half (the caller decides exactly).
G17_HD unsigned long long scaled_round(unsigned long long m, int e, int k) {
    const Pow10Entry& p = pow10(k);
    // 192-bit product m * (hi:lo) = W2:W1:W0
    const unsigned long long l0 = m * p.lo, l1 = mulhi64(m, p.lo);
    const unsigned long long h0 = m * p.hi, h1 = mulhi64(m, p.hi);
    const unsigned long long W0 = l0;
    const unsigned long long W1 = l1 + h0;
    const unsigned long long W2 = h1 + (W1 < l1 ? 1ull : 0ull);
    // t = product * 2^(e + p.e): integer part above bit S, S = -(e + p.e) in [64, 128)
    const int S = -(e + p.e);
    unsigned long long ti, fhi, flo;  // integer part; fraction = fhi:flo (S bits, left-aligned to 128)
    if (S >= 128) {
        const int r = S - 128;
        ti = r ? (W2 >> r) : W2;
        fhi = r ? ((W2 << (64 - r)) | (W1 >> r)) : W1;
        flo = r ? ((W1 << (64 - r)) | (W0 >> r)) : W0;
    } else {
        const int r = S - 64;  // 0 < r < 64 in practice
        ti = (W2 << (64 - r)) | (W1 >> r);
        fhi = (W1 << (64 - r)) | (W0 >> r);
        flo = W0 << (64 - r);
    }
    // fraction F in [0, 1) as the 128-bit fixed point fhi:flo; the truncation of
    // the table entry makes the true fraction F + err, 0 <= err < m 2^-S
    const unsigned long long HALF = 1ull << 63;
    const bool above = fhi > HALF || (fhi == HALF && flo != 0);
    const bool exact_half = fhi == HALF && flo == 0;
    if (p.exact) {
        if (above || (exact_half && (ti & 1))) return ti + 1;
        return ti;
    }
    if (above) return ti + 1;  // true fraction >= F > 1/2
    // below one half by more than the error bound (2^(53 + 128 - S) in fhi:flo units)?
    const int sh = 128 - S;
    const unsigned long long gap_hi = HALF - fhi - (flo ? 1 : 0);
    const bool far = (53 + sh >= 64) ? (gap_hi > (1ull << (53 + sh - 64))) : (gap_hi > 0);
    if (far && !exact_half) return ti;
    // near the midpoint: decide exactly (never reached for typical data)
    return ti | 0x8000000000000000ull;  // flag: caller resolves
}

// Writes "%.17g" of v into out (at least 25 bytes); returns the length.
G17_HD int format(double v, char* out) {
    unsigned long long bits;
#if defined(__CUDA_ARCH__)
    bits = (unsigned long long)__double_as_longlong(v);
#else
    __builtin_memcpy(&bits, &v, 8);
#endif
    int n = 0;
    const bool neg = bits >> 63;
    const int be = (int)((bits >> 52) & 0x7ff);
    unsigned long long frac = bits & ((1ull << 52) - 1);
    if (be == 0x7ff) {
        if (neg) out[n++] = '-';
        if (frac) {
            out[n++] = 'n';
            out[n++] = 'a';
            out[n++] = 'n';
        } else {
            out[n++] = 'i';
            out[n++] = 'n';
            out[n++] = 'f';
        }
        return n;
    }
    if (neg) out[n++] = '-';
    if (be == 0 && frac == 0) {
        out[n++] = '0';
        return n;
    }
    // |v| = m 2^e with m normalised to 53 bits
    unsigned long long m;
    int e;
    if (be) {
        m = frac | (1ull << 52);
        e = be - 1075;
    } else {
        const int lz = clz64(frac) - 11;  // shift to put the leading bit at 52
        m = frac << lz;
        e = -1074 - lz;
    }
    const int e2 = e + 52;                 // floor(log2 |v|)
    int X = (e2 * 78913) >> 18;            // floor(e2 log10 2): 10^X <= |v| < 2 10^(X+1)
    unsigned long long D = 0;
    for (int pass = 0; pass < 2; ++pass) {
        D = scaled_round(m, e, 16 - X);
        if (D >> 63) {  // near-midpoint: exact comparison with (2 floor + 1)/2
            const unsigned long long fl = D & 0x7fffffffffffffffull;
            const int c = cmp_midpoint(m, e, fl, X - 16);
            D = (c > 0 || (c == 0 && (fl & 1))) ? fl + 1 : fl;
        }
        if (D < 100000000000000000ull) break;
        ++X;  // rounded up to 10^17 or the estimate was one decade low
    }
    // 17 digits of D
    char dg[17];
    {
        unsigned long long q = D / 100000000ull;
        uint32_t lo8 = (uint32_t)(D - q * 100000000ull);
        const uint32_t top = (uint32_t)(q / 100000000ull);
        uint32_t mid8 = (uint32_t)(q - (unsigned long long)top * 100000000ull);
        for (int i = 16; i >= 9; --i) {
            dg[i] = (char)('0' + lo8 % 10);
            lo8 /= 10;
        }
        for (int i = 8; i >= 1; --i) {
            dg[i] = (char)('0' + mid8 % 10);
            mid8 /= 10;
        }
        dg[0] = (char)('0' + top);
    }
    int nd = 17;
    while (nd > 1 && dg[nd - 1] == '0') --nd;
    if (X >= -4 && X < 17) {
        if (X >= 0) {
            for (int i = 0; i <= X; ++i) out[n++] = i < nd ? dg[i] : '0';
            if (nd > X + 1) {
                out[n++] = '.';
                for (int i = X + 1; i < nd; ++i) out[n++] = dg[i];
            }
        } else {
            out[n++] = '0';
            out[n++] = '.';
            for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
            for (int i = 0; i < nd; ++i) out[n++] = dg[i];
        }
    } else {
        out[n++] = dg[0];
        if (nd > 1) {
            out[n++] = '.';
            for (int i = 1; i < nd; ++i) out[n++] = dg[i];
        }
        out[n++] = 'e';
        int x = X;
        if (x < 0) {
            out[n++] = '-';
            x = -x;
        } else {
            out[n++] = '+';
        }
        if (x >= 100) {
            out[n++] = (char)('0' + x / 100);
            x %= 100;
            out[n++] = (char)('0' + x / 10);
            out[n++] = (char)('0' + x % 10);
        } else {
            out[n++] = (char)('0' + x / 10);
            out[n++] = (char)('0' + x % 10);
        }
    }
    return n;
}

}  // namespace g17
}  // namespace petto_b200
