// apo_device.cuh -- device primitives shared by every APO kernel.
//
//  * keyed RNG: the reference's fmix64 chain (rng.py:79-111,
//    numba_backend.py:52-71), reproduced bit for bit;
//  * glibc-compatible exp: the reference evaluates the neighbour weight
//    exp(-|f_km/(f_kp+eps)|) (core.py:253-255, numba_backend.py:228,249) with
//    glibc's exp.  This is glibc 2.39's table-driven algorithm (N=128,
//    degree-5 polynomial, the x86-64 FMA build's contraction pattern), so
//    the device weight equals the CPU weight bit for bit.  The 2^(k/128)
//    table is derived with 300-bit arithmetic by tools/gen_exp_table.py;
//    tests/test_exp_port.py checks the C twin of this routine against the
//    host libm on 10^7 inputs;
//  * order-preserving 64-bit sort keys for fp64 fitness (numpy stable
//    argsort semantics: -0.0 == +0.0, NaN last).
//
// Oracle-mode translation units are compiled with --fmad=false: the
// reference never fuses a multiply-add, so neither may we.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cmath>

namespace apo {

constexpr uint64_t kH0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMul1 = 0xFF51AFD7ED558CCDULL;
constexpr uint64_t kMul2 = 0xC4CEB9FE1A85EC53ULL;
constexpr double kInv2p53 = 1.0 / 9007199254740992.0;

// Draw-slot layout: core.py:18-47
constexpr uint64_t kSlotDecision = 0, kSlotSign = 1, kSlotMaskSize = 2, kSlotMagnitude = 3, kSlotForage = 4,
                   kSlotPartner = 5, kVectorBase = 8, kMaskBase = 1ULL << 32, kPairsBase = 1ULL << 33;
constexpr uint64_t kCoordinator = 0xFFFFFFFFFFFFFFFFULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 33;
    z *= kMul1;
    z ^= z >> 33;
    z *= kMul2;
    z ^= z >> 33;
    return z;
}

__host__ __device__ __forceinline__ uint64_t stream_base(uint64_t seed, uint64_t iteration, uint64_t individual) {
    uint64_t h = mix64(kH0 ^ seed);
    h = mix64(h ^ iteration);
    return mix64(h ^ individual);
}

__host__ __device__ __forceinline__ double uniform(uint64_t base, uint64_t counter) {
    return (double)(mix64(base ^ counter) >> 11) * kInv2p53;
}

// ---------------------------------------------------------------------------
// Production RNG: Philox4x32-10 (Salmon et al., SC'11), one counter-based
// stream per (seed, iteration, protozoon): key = seed, counter block =
// (slot lo, slot hi, protozoon, iteration); the draw is the top 53 bits of
// the first two output words.  Slots are the reference's draw-slot layout
// (core.py:18-47), so every draw keeps its meaning; only the bits differ.
enum RngMode : int { RNG_KEYED = 0, RNG_PHILOX = 1, RNG_TABLE = 2 };

// Scripted draws (APO_RNG_TABLE, include/apo_b200.h apo_draw_table): the stream's `seed` word carries
// the device address of the table; a draw is looked up by (individual, counter) in entries sorted by
// that pair.  A draw the table does not hold records the first such address in miss[1..2], sets
// miss[0] and reads 0.0 (so every index derived from it stays in range); the host then fails the call
// (the reference's ScriptedStream fails on any unscripted read, tests/test_acceptance.py:50-80).
struct DrawTable {
    long long n;
    const unsigned long long* individual;
    const unsigned long long* counter;
    const double* value;
    unsigned long long* miss;
};

__host__ __device__ __forceinline__ void philox_mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#ifdef __CUDA_ARCH__
    hi = __umulhi(a, b);
    lo = a * b;
#else
    const uint64_t p = (uint64_t)a * (uint64_t)b;
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
#endif
}

__host__ __device__ inline void philox4x32_10_block(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        uint32_t hi0, lo0, hi1, lo1;
        philox_mulhilo(0xD2511F53u, c[0], hi0, lo0);
        philox_mulhilo(0xCD9E8D57u, c[2], hi1, lo1);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__host__ __device__ inline uint64_t philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                  uint32_t k1) {
    uint32_t c[4] = {c0, c1, c2, c3};
    philox4x32_10_block(c, k0, k1);
    return ((uint64_t)c[0] << 32) | c[1];
}

// Per-protozoon stream key for either generator.  uniform(Key, counter) is
// the only draw primitive the kernels use.
// Key.c of a scripted-draw key: lets the one out-of-line draw function tell the table from Philox
// without a mode argument (Philox keys carry the iteration there, < 2^31 on every entry point).
constexpr uint32_t kTableMark = 0xFFFFFFFFu;

struct Key {
    uint64_t a;   // keyed: the fmix64 stream base; philox: the seed
    uint32_t b;   // philox: protozoon (folded to 32 bits; the coordinator maps above 2^31)
    uint32_t c;   // philox: iteration
    int mode;
};

__host__ __device__ __forceinline__ Key stream_key(int mode, uint64_t seed, uint64_t iteration, uint64_t individual) {
    Key k;
    k.mode = mode;
    if (mode == RNG_PHILOX) {
        k.a = seed;
        k.b = (uint32_t)individual ^ ((uint32_t)(individual >> 32) * 0x9E3779B9u);
        k.c = (uint32_t)iteration;
    } else if (mode == RNG_TABLE) {  // a = table address, b = the individual (the script is one iteration)
        k.a = seed;
        k.b = individual == kCoordinator ? 0xFFFFFFFFu : (uint32_t)individual;  // protozoa are < 2^31
        k.c = kTableMark;
    } else {
        k.a = stream_base(seed, iteration, individual);
        k.b = k.c = 0;
    }
    return k;
}

__host__ __device__ __forceinline__ double philox_draw(uint64_t seed, uint32_t b, uint32_t c, uint64_t counter) {
    return (double)(philox4x32_10((uint32_t)counter, (uint32_t)(counter >> 32), b, c, (uint32_t)seed,
                                  (uint32_t)(seed >> 32)) >> 11) * kInv2p53;
}

#ifdef __CUDA_ARCH__
// Out of line where keyed draws dominate (a call site in the keyed loops is cheaper than 10 rounds
// inlined); the Philox builds of the hot kernels (APO_PHILOX_VARIANT) inline it.
#if defined(APO_PHILOX_VARIANT) && !defined(APO_PHILOX_CALL)
__device__ __forceinline__ double philox_uniform(uint64_t seed, uint32_t b, uint32_t c, uint64_t counter) {
#else
__device__ __noinline__ double philox_uniform(uint64_t seed, uint32_t b, uint32_t c, uint64_t counter) {
#endif
    return philox_draw(seed, b, c, counter);
}
#ifdef APO_RNG_TABLE_ENABLED
__device__ __forceinline__ double table_draw(uint64_t table, uint64_t individual, uint64_t counter) {
    const DrawTable* T = reinterpret_cast<const DrawTable*>(table);
    long long lo = 0, hi = T->n;  // first entry >= (individual, counter)
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        const unsigned long long mi = T->individual[mid], mc = T->counter[mid];
        if (mi < individual || (mi == individual && mc < counter)) lo = mid + 1;
        else hi = mid;
    }
    if (lo < T->n && T->individual[lo] == individual && T->counter[lo] == counter) return T->value[lo];
    if (atomicCAS(&T->miss[0], 0ull, 1ull) == 0ull) {
        T->miss[1] = individual;
        T->miss[2] = counter;
    }
    return 0.0;
}
#endif
#endif

// Scripted keys (c == kTableMark) are only read by kernels built with APO_RNG_TABLE_ENABLED -- their
// own instantiations in apo_update_scripted.cu: any table code in the keyed kernels, even on a branch
// they never take, measured +1.5-9% on the C4 update (it shifts ptxas' register allocation).
__host__ __device__ __forceinline__ double uniform(const Key& k, uint64_t counter) {
#if defined(APO_RNG_KEYED_ONLY) && defined(__CUDA_ARCH__)
    return uniform(k.a, counter);  // keyed builds: the hot kernels carry no Philox call site
#endif
    if (k.mode == RNG_KEYED) return uniform(k.a, counter);
#ifdef __CUDA_ARCH__
#ifdef APO_RNG_TABLE_ENABLED
    if (k.c == kTableMark) return table_draw(k.a, k.b == 0xFFFFFFFFu ? kCoordinator : (uint64_t)k.b, counter);
#endif
    return philox_uniform(k.a, k.b, k.c, counter);
#else
    return k.c == kTableMark ? 0.0 : philox_draw(k.a, k.b, k.c, counter);  // host: the table is device memory
#endif
}

// ---------------------------------------------------------------------------
// glibc exp (sysdeps/ieee754/dbl-64/e_exp.c algorithm, FMA build).

#define APO_EXP_TABLE { \
    0x0000000000000000ULL, 0x3ff0000000000000ULL, 0x3c9b3b4f1a88bf6eULL, 0x3feff63da9fb3335ULL, \
    0xbc7160139cd8dc5dULL, 0x3fefec9a3e778061ULL, 0xbc905e7a108766d1ULL, 0x3fefe315e86e7f85ULL, \
    0x3c8cd2523567f613ULL, 0x3fefd9b0d3158574ULL, 0xbc8bce8023f98efaULL, 0x3fefd06b29ddf6deULL, \
    0x3c60f74e61e6c861ULL, 0x3fefc74518759bc8ULL, 0x3c90a3e45b33d399ULL, 0x3fefbe3ecac6f383ULL, \
    0x3c979aa65d837b6dULL, 0x3fefb5586cf9890fULL, 0x3c8eb51a92fdeffcULL, 0x3fefac922b7247f7ULL, \
    0x3c3ebe3d702f9cd1ULL, 0x3fefa3ec32d3d1a2ULL, 0xbc6a033489906e0bULL, 0x3fef9b66affed31bULL, \
    0xbc9556522a2fbd0eULL, 0x3fef9301d0125b51ULL, 0xbc5080ef8c4eea55ULL, 0x3fef8abdc06c31ccULL, \
    0xbc91c923b9d5f416ULL, 0x3fef829aaea92de0ULL, 0x3c80d3e3e95c55afULL, 0x3fef7a98c8a58e51ULL, \
    0xbc801b15eaa59348ULL, 0x3fef72b83c7d517bULL, 0xbc8f1ff055de323dULL, 0x3fef6af9388c8deaULL, \
    0x3c8b898c3f1353bfULL, 0x3fef635beb6fcb75ULL, 0xbc96d99c7611eb26ULL, 0x3fef5be084045cd4ULL, \
    0x3c9aecf73e3a2f60ULL, 0x3fef54873168b9aaULL, 0xbc8fe782cb86389dULL, 0x3fef4d5022fcd91dULL, \
    0x3c8a6f4144a6c38dULL, 0x3fef463b88628cd6ULL, 0x3c807a05b0e4047dULL, 0x3fef3f49917ddc96ULL, \
    0x3c968efde3a8a894ULL, 0x3fef387a6e756238ULL, 0x3c875e18f274487dULL, 0x3fef31ce4fb2a63fULL, \
    0x3c80472b981fe7f2ULL, 0x3fef2b4565e27cddULL, 0xbc96b87b3f71085eULL, 0x3fef24dfe1f56381ULL, \
    0x3c82f7e16d09ab31ULL, 0x3fef1e9df51fdee1ULL, 0xbc3d219b1a6fbffaULL, 0x3fef187fd0dad990ULL, \
    0x3c8b3782720c0ab4ULL, 0x3fef1285a6e4030bULL, 0x3c6e149289cecb8fULL, 0x3fef0cafa93e2f56ULL, \
    0x3c834d754db0abb6ULL, 0x3fef06fe0a31b715ULL, 0x3c864201e2ac744cULL, 0x3fef0170fc4cd831ULL, \
    0x3c8fdd395dd3f84aULL, 0x3feefc08b26416ffULL, 0xbc86a3803b8e5b04ULL, 0x3feef6c55f929ff1ULL, \
    0xbc924aedcc4b5068ULL, 0x3feef1a7373aa9cbULL, 0xbc9907f81b512d8eULL, 0x3feeecae6d05d866ULL, \
    0xbc71d1e83e9436d2ULL, 0x3feee7db34e59ff7ULL, 0xbc991919b3ce1b15ULL, 0x3feee32dc313a8e5ULL, \
    0x3c859f48a72a4c6dULL, 0x3feedea64c123422ULL, 0xbc9312607a28698aULL, 0x3feeda4504ac801cULL, \
    0xbc58a78f4817895bULL, 0x3feed60a21f72e2aULL, 0xbc7c2c9b67499a1bULL, 0x3feed1f5d950a897ULL, \
    0x3c4363ed60c2ac11ULL, 0x3feece086061892dULL, 0x3c9666093b0664efULL, 0x3feeca41ed1d0057ULL, \
    0x3c6ecce1daa10379ULL, 0x3feec6a2b5c13cd0ULL, 0x3c93ff8e3f0f1230ULL, 0x3feec32af0d7d3deULL, \
    0x3c7690cebb7aafb0ULL, 0x3feebfdad5362a27ULL, 0x3c931dbdeb54e077ULL, 0x3feebcb299fddd0dULL, \
    0xbc8f94340071a38eULL, 0x3feeb9b2769d2ca7ULL, 0xbc87deccdc93a349ULL, 0x3feeb6daa2cf6642ULL, \
    0xbc78dec6bd0f385fULL, 0x3feeb42b569d4f82ULL, 0xbc861246ec7b5cf6ULL, 0x3feeb1a4ca5d920fULL, \
    0x3c93350518fdd78eULL, 0x3feeaf4736b527daULL, 0x3c7b98b72f8a9b05ULL, 0x3feead12d497c7fdULL, \
    0x3c9063e1e21c5409ULL, 0x3feeab07dd485429ULL, 0x3c34c7855019c6eaULL, 0x3feea9268a5946b7ULL, \
    0x3c9432e62b64c035ULL, 0x3feea76f15ad2148ULL, 0xbc8ce44a6199769fULL, 0x3feea5e1b976dc09ULL, \
    0xbc8c33c53bef4da8ULL, 0x3feea47eb03a5585ULL, 0xbc845378892be9aeULL, 0x3feea34634ccc320ULL, \
    0xbc93cedd78565858ULL, 0x3feea23882552225ULL, 0x3c5710aa807e1964ULL, 0x3feea155d44ca973ULL, \
    0xbc93b3efbf5e2228ULL, 0x3feea09e667f3bcdULL, 0xbc6a12ad8734b982ULL, 0x3feea012750bdabfULL, \
    0xbc6367efb86da9eeULL, 0x3fee9fb23c651a2fULL, 0xbc80dc3d54e08851ULL, 0x3fee9f7df9519484ULL, \
    0xbc781f647e5a3ecfULL, 0x3fee9f75e8ec5f74ULL, 0xbc86ee4ac08b7db0ULL, 0x3fee9f9a48a58174ULL, \
    0xbc8619321e55e68aULL, 0x3fee9feb564267c9ULL, 0x3c909ccb5e09d4d3ULL, 0x3feea0694fde5d3fULL, \
    0xbc7b32dcb94da51dULL, 0x3feea11473eb0187ULL, 0x3c94ecfd5467c06bULL, 0x3feea1ed0130c132ULL, \
    0x3c65ebe1abd66c55ULL, 0x3feea2f336cf4e62ULL, 0xbc88a1c52fb3cf42ULL, 0x3feea427543e1a12ULL, \
    0xbc9369b6f13b3734ULL, 0x3feea589994cce13ULL, 0xbc805e843a19ff1eULL, 0x3feea71a4623c7adULL, \
    0xbc94d450d872576eULL, 0x3feea8d99b4492edULL, 0x3c90ad675b0e8a00ULL, 0x3feeaac7d98a6699ULL, \
    0x3c8db72fc1f0eab4ULL, 0x3feeace5422aa0dbULL, 0xbc65b6609cc5e7ffULL, 0x3feeaf3216b5448cULL, \
    0x3c7bf68359f35f44ULL, 0x3feeb1ae99157736ULL, 0xbc93091fa71e3d83ULL, 0x3feeb45b0b91ffc6ULL, \
    0xbc5da9b88b6c1e29ULL, 0x3feeb737b0cdc5e5ULL, 0xbc6c23f97c90b959ULL, 0x3feeba44cbc8520fULL, \
    0xbc92434322f4f9aaULL, 0x3feebd829fde4e50ULL, 0xbc85ca6cd7668e4bULL, 0x3feec0f170ca07baULL, \
    0x3c71affc2b91ce27ULL, 0x3feec49182a3f090ULL, 0x3c6dd235e10a73bbULL, 0x3feec86319e32323ULL, \
    0xbc87c50422622263ULL, 0x3feecc667b5de565ULL, 0x3c8b1c86e3e231d5ULL, 0x3feed09bec4a2d33ULL, \
    0xbc91bbd1d3bcbb15ULL, 0x3feed503b23e255dULL, 0x3c90cc319cee31d2ULL, 0x3feed99e1330b358ULL, \
    0x3c8469846e735ab3ULL, 0x3feede6b5579fdbfULL, 0xbc82dfcd978e9db4ULL, 0x3feee36bbfd3f37aULL, \
    0x3c8c1a7792cb3387ULL, 0x3feee89f995ad3adULL, 0xbc907b8f4ad1d9faULL, 0x3feeee07298db666ULL, \
    0xbc55c3d956dcaebaULL, 0x3feef3a2b84f15fbULL, 0xbc90a40e3da6f640ULL, 0x3feef9728de5593aULL, \
    0xbc68d6f438ad9334ULL, 0x3feeff76f2fb5e47ULL, 0xbc91eee26b588a35ULL, 0x3fef05b030a1064aULL, \
    0x3c74ffd70a5fddcdULL, 0x3fef0c1e904bc1d2ULL, 0xbc91bdfbfa9298acULL, 0x3fef12c25bd71e09ULL, \
    0x3c736eae30af0cb3ULL, 0x3fef199bdd85529cULL, 0x3c8ee3325c9ffd94ULL, 0x3fef20ab5fffd07aULL, \
    0x3c84e08fd10959acULL, 0x3fef27f12e57d14bULL, 0x3c63cdaf384e1a67ULL, 0x3fef2f6d9406e7b5ULL, \
    0x3c676b2c6c921968ULL, 0x3fef3720dcef9069ULL, 0xbc808a1883ccb5d2ULL, 0x3fef3f0b555dc3faULL, \
    0xbc8fad5d3ffffa6fULL, 0x3fef472d4a07897cULL, 0xbc900dae3875a949ULL, 0x3fef4f87080d89f2ULL, \
    0x3c74a385a63d07a7ULL, 0x3fef5818dcfba487ULL, 0xbc82919e2040220fULL, 0x3fef60e316c98398ULL, \
    0x3c8e5a50d5c192acULL, 0x3fef69e603db3285ULL, 0x3c843a59ac016b4bULL, 0x3fef7321f301b460ULL, \
    0xbc82d52107b43e1fULL, 0x3fef7c97337b9b5fULL, 0xbc892ab93b470dc9ULL, 0x3fef864614f5a129ULL, \
    0x3c74b604603a88d3ULL, 0x3fef902ee78b3ff6ULL, 0x3c83c5ec519d7271ULL, 0x3fef9a51fbc74c83ULL, \
    0xbc8ff7128fd391f0ULL, 0x3fefa4afa2a490daULL, 0xbc8dae98e223747dULL, 0x3fefaf482d8e67f1ULL, \
    0x3c8ec3bc41aa2008ULL, 0x3fefba1bee615a27ULL, 0x3c842b94c3a9eb32ULL, 0x3fefc52b376bba97ULL, \
    0x3c8a64a931d185eeULL, 0x3fefd0765b6e4540ULL, 0xbc8e37bae43be3edULL, 0x3fefdbfdad9cbe14ULL, \
    0x3c77893b4d91cd9dULL, 0x3fefe7c1819e90d8ULL, 0x3c5305c14160cc89ULL, 0x3feff3c22b8f71f1ULL, \
}
__constant__ uint64_t kExpTab[256] = APO_EXP_TABLE;
static const uint64_t kExpTabHost[256] = APO_EXP_TABLE;

#ifdef __CUDA_ARCH__
#define APO_DMUL(a, b) __dmul_rn(a, b)
#define APO_DADD(a, b) __dadd_rn(a, b)
#define APO_DSUB(a, b) __dsub_rn(a, b)
#define APO_DDIV(a, b) __ddiv_rn(a, b)
#define APO_FMA(a, b, c) __fma_rn(a, b, c)
#define APO_EXPTAB kExpTab
#else
#define APO_DMUL(a, b) ((a) * (b))
#define APO_DADD(a, b) ((a) + (b))
#define APO_DSUB(a, b) ((a) - (b))
#define APO_DDIV(a, b) ((a) / (b))
#define APO_FMA(a, b, c) fma(a, b, c)
#define APO_EXPTAB kExpTabHost
#endif

__host__ __device__ __forceinline__ double bits_to_double(uint64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double f;
    __builtin_memcpy(&f, &b, 8);
    return f;
#endif
}
__host__ __device__ __forceinline__ uint64_t double_to_bits(double f) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(f);
#else
    uint64_t b;
    __builtin_memcpy(&b, &f, 8);
    return b;
#endif
}

__host__ __device__ __forceinline__ double exp_glibc_special(double tmp, uint64_t sbits, uint64_t ki) {
    // glibc's specialcase() is reached for |x| >= 512; it is evaluated
    // without contraction (matches the host libm bit for bit).
    double scale, y;
    if ((ki & 0x80000000ULL) == 0) {
        sbits -= 1009ULL << 52;
        scale = bits_to_double(sbits);
        y = APO_DMUL(0x1p1009, APO_DADD(scale, APO_DMUL(scale, tmp)));
        return y;
    }
    sbits += 1022ULL << 52;
    scale = bits_to_double(sbits);
    y = APO_DADD(scale, APO_DMUL(scale, tmp));
    if (y < 1.0) {
        double lo = APO_DADD(APO_DSUB(scale, y), APO_DMUL(scale, tmp));
        double hi = APO_DADD(1.0, y);
        lo = APO_DADD(APO_DADD(APO_DSUB(1.0, hi), y), lo);
        y = APO_DSUB(APO_DADD(hi, lo), 1.0);
        if (y == 0.0) y = 0.0;
    }
    return APO_DMUL(0x1p-1022, y);
}

__host__ __device__ __forceinline__ double exp_glibc(double x) {
    const double kInvLn2N = 0x1.71547652b82fep0 * 128.0, kShift = 0x1.8p52;
    const double kNegLn2hiN = -0x1.62e42fefa0000p-8, kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3, C4 = 0x1.55555cf172b91p-5,
                 C5 = 0x1.1111167a4d017p-7;
    uint64_t ux = double_to_bits(x);
    uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if (abstop - 0x3c9u >= 0x80000000u) return APO_DADD(1.0, x);  // |x| < 2^-54
        if (abstop >= 0x409u) {                                         // |x| >= 1024
            if (ux == 0xfff0000000000000ULL) return 0.0;
            if (abstop >= 0x7ffu) return APO_DADD(1.0, x);
            return (ux >> 63) ? 0.0 : bits_to_double(0x7ff0000000000000ULL);
        }
        abstop = 0;  // large |x|: special-cased below
    }
    double z = APO_DMUL(kInvLn2N, x);
    double kd = APO_DADD(z, kShift);
    uint64_t ki = double_to_bits(kd);
    kd = APO_DSUB(kd, kShift);
    double r = APO_FMA(kd, kNegLn2loN, APO_FMA(kd, kNegLn2hiN, x));
    uint32_t idx = 2u * (uint32_t)(ki % 128u);
    uint64_t top = ki << 45;
    double tail = bits_to_double(APO_EXPTAB[idx]);
    uint64_t sbits = APO_EXPTAB[idx + 1] + top;
    double r2 = APO_DMUL(r, r);
    double tmp = APO_FMA(APO_DMUL(r2, r2), APO_FMA(r, C5, C4), APO_FMA(r2, APO_FMA(r, C3, C2), APO_DADD(tail, r)));
    if (abstop == 0) return exp_glibc_special(tmp, sbits, ki);
    double scale = bits_to_double(sbits);
    return APO_FMA(scale, tmp, scale);
}

// ---------------------------------------------------------------------------
// cos as glibc 2.39 computes it (sysdeps/ieee754/dbl-64/s_sin.c, __cos; the x86_64 FMA variant the
// host libm dispatches to on FMA-capable CPUs), so griewank (numba_backend.py:130, objectives.py:141)
// matches the reference bit for bit.  Table: glibc's __sincostab (tools/gen_cos_table.py).  Range
// reduction: |x| < 2.426 directly or from pi/2 - |x| in double-double; |x| < 105414350 by the 3-part
// Cody-Waite split of pi/2 (reduce_sincos).  Beyond that glibc uses a multi-precision reduction
// (__branred) that is not ported: CUDA's cos is used there (|x| >= 1e8 needs bounds far outside any
// benchmark's).  Every multiply-add below is the fused operation GCC emits for glibc's __cos_fma.
#include "apo_cos_glibc.h"
__device__ const uint64_t kSinCosTab[440] = APO_SINCOS_TABLE;  // divergent indices: global (L1), not __constant__
static const uint64_t kSinCosTabHost[440] = APO_SINCOS_TABLE;
#ifdef __CUDA_ARCH__
#define APO_SCTAB(i) bits_to_double(__ldg(reinterpret_cast<const unsigned long long*>(kSinCosTab) + (i)))
#else
#define APO_SCTAB(i) bits_to_double(kSinCosTabHost[i])
#endif

__host__ __device__ __forceinline__ double glibc_do_cos(double x, double dx) {
    const double big = 0x1.8p45, sn3 = -0x1.5555555555515p-3, sn5 = 0x1.11110e829872fp-7, cs2 = 0.5,
                 cs4 = -0x1.5555555555535p-5, cs6 = 0x1.6c16bedd9e239p-10;
    if (x < 0) dx = -dx;
    const double ux = APO_DADD(big, fabs(x));
    x = APO_DADD(APO_DSUB(fabs(x), APO_DSUB(ux, big)), dx);
    const double xx = APO_DMUL(x, x);
    const double s = APO_FMA(APO_DMUL(x, xx), APO_FMA(xx, sn5, sn3), x);
    const double c = APO_DMUL(xx, APO_FMA(xx, APO_FMA(xx, cs6, cs4), cs2));
    const int k = (int)(uint32_t)double_to_bits(ux) << 2;
    const double sn = APO_SCTAB(k), ssn = APO_SCTAB(k + 1), cs = APO_SCTAB(k + 2), ccs = APO_SCTAB(k + 3);
    const double cor = APO_FMA(-sn, s, APO_FMA(-cs, c, APO_FMA(-s, ssn, ccs)));
    return APO_DADD(cs, cor);
}

__host__ __device__ __forceinline__ double glibc_do_sin(double x, double dx) {
    const double big = 0x1.8p45, sn3 = -0x1.5555555555515p-3, sn5 = 0x1.11110e829872fp-7, cs2 = 0.5,
                 cs4 = -0x1.5555555555535p-5, cs6 = 0x1.6c16bedd9e239p-10;
    const double xold = x;
    if (fabs(x) < 0.126) {  // TAYLOR_SIN(x*x, x, dx)
        const double s1 = -0x1.5555555555555p-3, s2 = 0x1.1111111110ecep-7, s3 = -0x1.a01a019db08b8p-13,
                     s4 = 0x1.71de27b9a7ed9p-19, s5 = -0x1.addffc2fcdf59p-26;
        const double xx = APO_DMUL(x, x);
        const double p = APO_FMA(APO_FMA(APO_FMA(APO_FMA(s5, xx, s4), xx, s3), xx, s2), xx, s1);
        const double t = APO_FMA(APO_FMA(p, x, -APO_DMUL(0.5, dx)), xx, dx);
        return APO_DADD(x, t);
    }
    if (x <= 0) dx = -dx;
    const double ux = APO_DADD(big, fabs(x));
    x = APO_DSUB(fabs(x), APO_DSUB(ux, big));
    const double xx = APO_DMUL(x, x);
    const double s = APO_DADD(x, APO_FMA(APO_DMUL(x, xx), APO_FMA(xx, sn5, sn3), dx));
    const double c = APO_FMA(x, dx, APO_DMUL(xx, APO_FMA(xx, APO_FMA(xx, cs6, cs4), cs2)));
    const int k = (int)(uint32_t)double_to_bits(ux) << 2;
    const double sn = APO_SCTAB(k), ssn = APO_SCTAB(k + 1), cs = APO_SCTAB(k + 2), ccs = APO_SCTAB(k + 3);
    const double cor = APO_FMA(cs, s, APO_FMA(-sn, c, APO_FMA(s, ccs, ssn)));
    return copysign(APO_DADD(sn, cor), xold);
}

__host__ __device__ __forceinline__ double cos_glibc(double x) {
    const uint32_t k = (uint32_t)(double_to_bits(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) return 1.0;                      // |x| < 2^-27
    if (k < 0x3feb6000u) return glibc_do_cos(x, 0.0);    // |x| < 0.855469
    if (k < 0x400368fdu) {                                // |x| < 2.426265: cos x = sin(pi/2 - |x|)
        const double hp0 = 0x1.921fb54442d18p0, hp1 = 0x1.1a62633145c07p-54;
        const double y = APO_DSUB(hp0, fabs(x));
        const double a = APO_DADD(y, hp1);
        return glibc_do_sin(a, APO_DADD(APO_DSUB(y, a), hp1));
    }
    if (k < 0x419921fbu) {                                // |x| < 105414350: reduce_sincos
        const double hpinv = 0x1.45f306dc9c883p-1, toint = 0x1.8p52, mp1 = 0x1.921fb58p0,
                     mp2 = -0x1.dde973cp-27, pp3 = -0x1.cb3b398p-55, pp4 = -0x1.d747f23e32ed7p-83;
        const double t = APO_FMA(x, hpinv, toint);
        const double xn = APO_DSUB(t, toint);
        const double y = APO_FMA(-xn, mp2, APO_FMA(-xn, mp1, x));
        int n = (int)((uint32_t)double_to_bits(t) & 3u);
        double t1 = APO_DMUL(xn, pp3);
        const double t2 = APO_DSUB(y, t1);
        double db = APO_DSUB(APO_DSUB(y, t2), t1);
        t1 = APO_DMUL(xn, pp4);
        const double b = APO_DSUB(t2, t1);
        db = APO_DADD(db, APO_DSUB(APO_DSUB(t2, b), t1));
        n += 1;
        const double r = (n & 1) ? glibc_do_cos(b, db) : glibc_do_sin(b, db);
        return (n & 2) ? -r : r;
    }
    if (k < 0x7ff00000u) return cos(x);  // __branred range: not ported (see above)
    return x - x;                        // inf, nan -> nan
}

// Neighbour influence weight exp(-|fa/(fb+eps)|): core.py:253-255.
__host__ __device__ __forceinline__ double rank_weight(double fa, double fb, double eps) {
    return exp_glibc(-fabs(APO_DDIV(fa, APO_DADD(fb, eps))));
}

// ---------------------------------------------------------------------------
// Order-preserving key: ascending doubles, -0.0 == +0.0, every NaN last.
__host__ __device__ __forceinline__ uint64_t sort_key(double f) {
    if (f != f) return 0xFFFFFFFFFFFFFFFFULL;
    if (f == 0.0) return 0x8000000000000000ULL;
    uint64_t b = double_to_bits(f);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__host__ __device__ __forceinline__ double key_to_double(uint64_t k) {
    if (k == 0xFFFFFFFFFFFFFFFFULL) return bits_to_double(0x7ff8000000000000ULL);
    return bits_to_double((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k);
}

}  // namespace apo
