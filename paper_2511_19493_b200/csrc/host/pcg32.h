// pcg32.h — PCG32 streams (host and device), rng.py:41-70 semantics.
//
// A stream is (state, inc).  make(seed, seq): inc = (seq << 1) | 1, state = 0,
// step, state += seed (mod 2^64), step.  The output function is the
// XSH-RR permutation of the OLD state.  Also provides the LCG jump-ahead the
// device uses to start a thread at an arbitrary position of a stream.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define RFX_HD __host__ __device__ __forceinline__
#else
#define RFX_HD static inline
#endif

enum { RFX_SEQ_TREE = 1, RFX_SEQ_FACTOR = 3, RFX_SEQ_PMAX = 4, RFX_SEQ_POWER = 5,
       RFX_SEQ_GROW = 7 };

#define RFX_PCG_MULT 6364136223846793005ULL

RFX_HD uint32_t rfx_pcg32_next(uint64_t* s)
{
    uint64_t old = s[0];
    s[0] = old * RFX_PCG_MULT + s[1];
    uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

RFX_HD void rfx_pcg32_make(int64_t seed, int64_t seq, uint64_t* s)
{
    s[0] = 0;
    s[1] = ((uint64_t)seq << 1) | 1ULL;
    rfx_pcg32_next(s);
    s[0] += (uint64_t)seed;
    rfx_pcg32_next(s);
}

RFX_HD uint32_t rfx_pcg32_bounded(uint64_t* s, uint32_t bound)
{
    uint64_t b = bound;
    uint64_t threshold = (0x100000000ULL - b) % b;
    for (;;) {
        uint64_t r = rfx_pcg32_next(s);
        if (r >= threshold) return (uint32_t)(r % b);
    }
}

// Advance the LCG state by `delta` steps in O(log delta) (Brown, "Random
// number generation with arbitrary strides").
RFX_HD void rfx_pcg32_advance(uint64_t* s, uint64_t delta)
{
    uint64_t cur_mult = RFX_PCG_MULT, cur_plus = s[1];
    uint64_t acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    s[0] = acc_mult * s[0] + acc_plus;
}
