// philox.cuh — counter-based Philox4x32-10 streams, host and device.
//
// Same stream derivation and draw semantics as the reference RngStream
// (proj/src/rng.cpp:9-94): key = splitmix64(seed); stream id =
// splitmix64(splitmix64(seed') ^ idx*0xA24BAED4963EE407 ^ fnv1a64(purpose));
// one 128-bit block per draw, indexed by a 64-bit draw counter. Because the
// generator is a pure function of (key, stream, counter), every GPU thread can
// produce any draw of any chain directly — no sequential state.
#pragma once

#include <stdint.h>

#include <cmath>

namespace dgb {

struct PhiloxKey {
    uint32_t k0, k1;  // key
    uint32_t s0, s1;  // stream words (counter words 2,3)
};

__host__ __device__ inline uint64_t splitmix64_step(uint64_t& state) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline uint64_t fnv1a64_host(const char* s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (; *s; ++s) {
        h ^= static_cast<unsigned char>(*s);
        h *= 0x100000001b3ull;
    }
    return h;
}

inline PhiloxKey make_philox_key(uint64_t master_seed, uint64_t stream_index, const char* purpose) {
    uint64_t s = master_seed;
    const uint64_t k = splitmix64_step(s);
    uint64_t id = splitmix64_step(s) ^ (stream_index * 0xA24BAED4963EE407ull) ^ fnv1a64_host(purpose);
    const uint64_t sid = splitmix64_step(id);
    return PhiloxKey{static_cast<uint32_t>(k), static_cast<uint32_t>(k >> 32),
                     static_cast<uint32_t>(sid), static_cast<uint32_t>(sid >> 32)};
}

struct Block4 {
    uint32_t w[4];
};

__host__ __device__ inline Block4 philox_block(const PhiloxKey& key, uint64_t counter) {
    uint32_t c0 = static_cast<uint32_t>(counter), c1 = static_cast<uint32_t>(counter >> 32);
    uint32_t c2 = key.s0, c3 = key.s1;
    uint32_t k0 = key.k0, k1 = key.k1;
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
#else
        const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
        const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
        const uint32_t lo0 = static_cast<uint32_t>(p0), hi0 = static_cast<uint32_t>(p0 >> 32);
        const uint32_t lo1 = static_cast<uint32_t>(p1), hi1 = static_cast<uint32_t>(p1 >> 32);
#endif
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return Block4{{c0, c1, c2, c3}};
}

__host__ __device__ inline uint64_t philox_u64(const PhiloxKey& key, uint64_t counter) {
    const Block4 b = philox_block(key, counter);
    return (static_cast<uint64_t>(b.w[1]) << 32) | b.w[0];
}

// uniform in (0,1): proj/src/rng.cpp:81-83 (bit-exact: integer -> double is exact)
__host__ __device__ inline double philox_uniform_open(const PhiloxKey& key, uint64_t counter) {
    return (static_cast<double>(philox_u64(key, counter) >> 11) + 0.5) * 0x1.0p-53;
}

// standard normal, Box-Muller cosine branch: proj/src/rng.cpp:85-94. The
// integer part is bit-exact; log/cos are CUDA's double-precision libm (<=1/2
// ulp class differences from glibc, measured in tests/test_gpu_rng.py).
__host__ __device__ inline double philox_normal(const PhiloxKey& key, uint64_t counter) {
    const Block4 b = philox_block(key, counter);
    const uint64_t w0 = (static_cast<uint64_t>(b.w[1]) << 32) | b.w[0];
    const uint64_t w1 = (static_cast<uint64_t>(b.w[3]) << 32) | b.w[2];
    const double u1 = (static_cast<double>(w0 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(w1 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    // cos of the rounded product 2*pi*u2, exactly as the reference: cospi(2*u2) would be
    // 5% faster but moves 0.1% of the normals by >1e-14 relative away from glibc's
    return r * cos(6.283185307179586476925286766559 * u2);
}

}  // namespace dgb
