// Keyed Gaussian noise that is bit-identical on the GPU and on the CPU.
//
// BASELINE configs 2 and 5 add i.i.d. Gaussian noise E scaled to a fraction
// of ||X||_F. The draws use the reference's keyed SplitMix (rng.hpp:11-36) on
// stream 0x4E01 at each entry's GLOBAL flat index (so the noise does not
// depend on the GPU count), and the Box-Muller map of rng.hpp:40-46. The one
// change: log and cos are evaluated by the fixed polynomial programs below,
// built only from correctly rounded +, -, *, / and sqrt with no fused
// multiply-add, instead of libm / libdevice (whose last bits differ between
// glibc and CUDA). The CPU restatement (oracle/cpkit_oracle.cpp, noise
// section) runs the same programs, so both produce the same bits, and the
// CPU baseline decomposes exactly the tensor the GPU decomposes.
//
// The noise scale needs ||X||^2 and ||E||^2 in an order that no GPU count
// changes: the slab is viewed as rows f' (all modes but the last) x columns j
// (last mode); block b of kNoiseBlocks consecutive-row blocks is summed
// sequentially per column, the blocks are summed per column in block order,
// and the columns in global j order. Each rank owns whole columns.
#pragma once
#include <cmath>
#include <cstdint>

namespace cpkit {
namespace noise {

constexpr int kNoiseBlocks = 256;
constexpr std::uint64_t kNoiseStream = 0x4E01;

#if defined(__CUDA_ARCH__)
#define CPK_NZ_MUL(a, b) __dmul_rn((a), (b))
#define CPK_NZ_ADD(a, b) __dadd_rn((a), (b))
#define CPK_NZ_SUB(a, b) __dadd_rn((a), -(b))
#define CPK_NZ_DIV(a, b) __ddiv_rn((a), (b))
#define CPK_NZ_SQRT(a) __dsqrt_rn(a)
#define CPK_NZ_FN __device__ __forceinline__
#else
#define CPK_NZ_MUL(a, b) ((a) * (b))
#define CPK_NZ_ADD(a, b) ((a) + (b))
#define CPK_NZ_SUB(a, b) ((a) - (b))
#define CPK_NZ_DIV(a, b) ((a) / (b))
#define CPK_NZ_SQRT(a) std::sqrt(a)
#define CPK_NZ_FN inline
#endif

CPK_NZ_FN std::uint64_t nz_mix64(std::uint64_t x) {  // rng.hpp:11-18
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
CPK_NZ_FN std::uint64_t nz_derive(std::uint64_t h, std::uint64_t v) {  // rng.hpp:20-23
    return nz_mix64(h ^ (v * 0xD6E8FEB86659FD93ull + 0xA0761D6478BD642Full));
}

// ln(u) for u in (0, 1] (normal numbers): u = m 2^e with m in [sqrt(1/2), sqrt(2)),
// ln m = 2 atanh(s), s = (m - 1) / (m + 1), |s| <= 0.1716, series to s^27.
CPK_NZ_FN double portable_log(double u) {
    std::uint64_t bits;
    static_assert(sizeof(double) == sizeof(std::uint64_t), "double is 64-bit");
#if defined(__CUDA_ARCH__)
    bits = static_cast<std::uint64_t>(__double_as_longlong(u));
#else
    __builtin_memcpy(&bits, &u, 8);
#endif
    int e = static_cast<int>((bits >> 52) & 0x7FF) - 1022;                  // u = m 2^e, m in [0.5, 1)
    bits = (bits & 0x000FFFFFFFFFFFFFull) | (static_cast<std::uint64_t>(1022) << 52);
    double m;
#if defined(__CUDA_ARCH__)
    m = __longlong_as_double(static_cast<long long>(bits));
#else
    __builtin_memcpy(&m, &bits, 8);
#endif
    if (m < 0x1.6a09e667f3bcdp-1) {  // sqrt(1/2)  // exact: doubling and the exponent shift are exact
        m = CPK_NZ_MUL(m, 2.0);
        e -= 1;
    }
    const double s = CPK_NZ_DIV(CPK_NZ_SUB(m, 1.0), CPK_NZ_ADD(m, 1.0));
    const double z = CPK_NZ_MUL(s, s);
    // 1 + z/3 + z^2/5 + ... + z^13/27 by Horner (coefficients fl(1/(2k+1)))
    constexpr double kl[14] = {0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3,
                               0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4,
                               0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
                               0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5,
                               0x1.47ae147ae147bp-5, 0x1.2f684bda12f68p-5};
    double p = kl[13];
    for (int i = 12; i >= 0; --i) p = CPK_NZ_ADD(CPK_NZ_MUL(p, z), kl[i]);
    const double lnm = CPK_NZ_MUL(CPK_NZ_MUL(2.0, s), p);
    const double de = static_cast<double>(e);
    constexpr double kLn2Hi = 0x1.62e42fee00000p-1;  // ln 2 split: e * hi is exact for |e| < 2^11
    constexpr double kLn2Lo = 0x1.a39ef35793c76p-33;
    return CPK_NZ_ADD(CPK_NZ_MUL(de, kLn2Hi), CPK_NZ_ADD(CPK_NZ_MUL(de, kLn2Lo), lnm));
}

// cos(2 pi u) for u in [0, 1): the quadrant comes from 4u exactly (u is a
// multiple of 2^-53), theta = r pi/2 in [0, pi/2), Taylor series of cos to
// theta^26 and of sin to theta^25 (coefficients fl(+-1/n!)).
CPK_NZ_FN double portable_cos_2pi(double u) {
    const double t = CPK_NZ_MUL(u, 4.0);  // exact
    const int k = static_cast<int>(t);
    const double r = CPK_NZ_SUB(t, static_cast<double>(k));  // exact
    const double th = CPK_NZ_MUL(r, 0x1.921fb54442d18p+0);  // pi/2
    const double z = CPK_NZ_MUL(th, th);
    constexpr double kc[14] = {0x1.0000000000000p+0,  -0x1.0000000000000p-1, 0x1.5555555555555p-5,
                               -0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-16,  -0x1.27e4fb7789f5cp-22,
                               0x1.1eed8eff8d898p-29,  -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45,
                               -0x1.6827863b97d97p-53, 0x1.e542ba4020225p-62,  -0x1.0ce396db7f853p-70,
                               0x1.f2cf01972f578p-80,  -0x1.88e85fc6a4e59p-89};
    constexpr double ks[13] = {0x1.0000000000000p+0,  -0x1.5555555555555p-3, 0x1.1111111111111p-7,
                               -0x1.a01a01a01a01ap-13, 0x1.71de3a556c734p-19,  -0x1.ae64567f544e4p-26,
                               0x1.6124613a86d09p-33,  -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49,
                               -0x1.2f49b46814157p-57, 0x1.71b8ef6dcf572p-66,  -0x1.761b413163819p-75,
                               0x1.3f3ccdd165fa9p-84};
    double cc = kc[13];
    for (int i = 12; i >= 0; --i) cc = CPK_NZ_ADD(CPK_NZ_MUL(cc, z), kc[i]);
    double ss = ks[12];
    for (int i = 11; i >= 0; --i) ss = CPK_NZ_ADD(CPK_NZ_MUL(ss, z), ks[i]);
    ss = CPK_NZ_MUL(ss, th);
    switch (k & 3) {
        case 0: return cc;   // cos(theta)
        case 1: return -ss;  // cos(pi/2 + theta)
        case 2: return -cc;  // cos(pi + theta)
        default: return ss;  // cos(3 pi/2 + theta)
    }
}

// rng::gaussian (rng.hpp:40-46) with the portable log / cos above.
CPK_NZ_FN double keyed_gaussian(std::uint64_t base /* derive(mix64(seed), stream) */, std::uint64_t gidx) {
    const std::uint64_t h = nz_derive(base, gidx);
    const double u1 = static_cast<double>((nz_derive(h, 1) >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(nz_derive(h, 2) >> 11) * 0x1.0p-53;
    return CPK_NZ_MUL(CPK_NZ_SQRT(CPK_NZ_MUL(-2.0, portable_log(u1))), portable_cos_2pi(u2));
}

}  // namespace noise
}  // namespace cpkit
