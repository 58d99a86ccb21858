// Host side of synk_gather_rows_inline: narrow a u64 index list to the u32
// kernel parameters and bounds-check it in the same pass. The list is read
// once by the calling thread (pinned or pageable memory); AVX-512 (vpcmpuq +
// vpmovqd, 16 indices per iteration) or AVX2 when the CPU has them, scalar
// otherwise.

#include <immintrin.h>

#include <cstdint>

namespace synk {

namespace {

uint32_t narrow_scalar(const uint64_t* in, uint64_t n, uint64_t limit, uint32_t* out) {
    uint32_t bad = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t v = in[i];
        const uint32_t ok = v < limit;
        bad |= ok ^ 1u;
        out[i] = ok ? static_cast<uint32_t>(v) : 0u;
    }
    return bad;
}

__attribute__((target("avx2"))) uint32_t narrow_avx2(const uint64_t* in, uint64_t n, uint64_t limit, uint32_t* out) {
    const __m256i sign = _mm256_set1_epi64x(static_cast<long long>(0x8000000000000000ull));
    const __m256i lim = _mm256_xor_si256(_mm256_set1_epi64x(static_cast<long long>(limit)), sign);
    const __m256i lo_dwords = _mm256_setr_epi32(0, 2, 4, 6, 0, 0, 0, 0);
    __m256i bad = _mm256_setzero_si256();
    uint64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + i));
        __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + i + 4));
        // unsigned v < limit  <=>  (limit ^ sign) > (v ^ sign) as signed
        const __m256i oka = _mm256_cmpgt_epi64(lim, _mm256_xor_si256(a, sign));
        const __m256i okb = _mm256_cmpgt_epi64(lim, _mm256_xor_si256(b, sign));
        bad = _mm256_or_si256(bad, _mm256_andnot_si256(_mm256_and_si256(oka, okb), _mm256_set1_epi64x(-1)));
        a = _mm256_and_si256(a, oka);  // an out-of-range index reads row 0
        b = _mm256_and_si256(b, okb);
        const __m128i na = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(a, lo_dwords));
        const __m128i nb = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(b, lo_dwords));
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + i), _mm256_set_m128i(nb, na));
    }
    uint32_t r = _mm256_testz_si256(bad, bad) ? 0u : 1u;
    return r | narrow_scalar(in + i, n - i, limit, out + i);
}

__attribute__((target("avx512f"))) uint32_t narrow_avx512(const uint64_t* in, uint64_t n, uint64_t limit,
                                                            uint32_t* out) {
    const __m512i lim = _mm512_set1_epi64(static_cast<long long>(limit));
    __mmask8 ok_all = 0xff;
    uint64_t i = 0;
    for (; i + 16 <= n; i += 16) {
        const __m512i a = _mm512_loadu_si512(in + i);
        const __m512i b = _mm512_loadu_si512(in + i + 8);
        const __mmask8 oka = _mm512_cmplt_epu64_mask(a, lim), okb = _mm512_cmplt_epu64_mask(b, lim);
        ok_all &= oka & okb;
        // vpmovqd: 8 x u64 -> 8 x u32 (an out-of-range index reads row 0)
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + i), _mm512_maskz_cvtepi64_epi32(oka, a));
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + i + 8), _mm512_maskz_cvtepi64_epi32(okb, b));
    }
    return (ok_all == 0xff ? 0u : 1u) | narrow_scalar(in + i, n - i, limit, out + i);
}

}  // namespace

// out[i] = in[i] < limit ? u32(in[i]) : 0; returns 1 when any index was out of
// range. limit <= 2^32.
uint32_t narrow_indices(const uint64_t* in, uint64_t n, uint64_t limit, uint32_t* out) {
    static const int isa = __builtin_cpu_supports("avx512f") ? 2 : __builtin_cpu_supports("avx2") ? 1 : 0;
    if (isa == 2) return narrow_avx512(in, n, limit, out);
    return isa == 1 ? narrow_avx2(in, n, limit, out) : narrow_scalar(in, n, limit, out);
}

}  // namespace synk
