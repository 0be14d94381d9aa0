// sgap_ingest.cuh -- Matrix Market -> CSR on the device.
//
// The reference parses coordinate Matrix Market text line by line in Python
// (matrices.py:144-212) and packs COO into CSR with a lexsort and
// np.add.reduceat (matrices.py:124-141).  Here the entry lines are indexed,
// tokenised and converted by one thread per line; tokens outside a strict
// grammar (or values the exact fast path cannot convert) are marked for the
// host, which applies Python's own int()/float() to just those lines, so the
// result and every error (message and line number) stay the reference's.
// Duplicates are summed in numpy's reduceat order (first element plus the
// pairwise sum of the rest), so values are bit-identical.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sgap {

enum MmStatus : unsigned char {
    kMmSkip = 0,    // blank or comment line
    kMmOk = 1,      // entry converted on the device
    kMmFields = 2,  // not exactly three tokens
    kMmNonNum = 3,  // a token is not a number (strict grammar, no exotic form)
    kMmRange = 4,   // coordinate outside the declared shape
    kMmHost = 5,    // needs Python's int()/float() (exotic token): the host checks the line
    kMmFloat = 6,   // entry whose plain-decimal value is off the exact fast path:
                    // converted on the host in one vectorised batch (tok_off/tok_len)
};

// Line starts (byte after each '\n', and byte 0) and "special" bytes that
// make str.splitlines()/str.split() differ from a '\n' / blank split: lone
// '\r', other control characters, non-ASCII.  Any special byte sends the
// whole body to the host parser.
__global__ void k_mm_line_flags(const unsigned char *__restrict__ t, long long len,
                                unsigned char *__restrict__ flag, int *__restrict__ special) {
    bool sp = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned char c = t[i];
        flag[i] = (i == 0 || t[i - 1] == '\n') ? 1 : 0;
        if (c >= 0x80 || (c < 0x20 && c != '\t' && c != '\n' && c != '\r') ||
            (c == '\r' && (i + 1 >= len || t[i + 1] != '\n')))
            sp = true;
    }
    if (__any_sync(0xffffffffu, sp) && (threadIdx.x & 31) == 0) atomicOr(special, 1);
}

__device__ __forceinline__ bool mm_space(unsigned char c) { return c == ' ' || c == '\t' || c == '\r'; }
__device__ __forceinline__ bool mm_digit(unsigned char c) { return c >= '0' && c <= '9'; }

// [+-]?[0-9]{1,18}: 0 ok, 1 anything else (Python may still accept it:
// underscores, unicode digits, huge values -> the host decides)
__device__ __forceinline__ int mm_int(const unsigned char *s, const unsigned char *e, long long &out) {
    bool neg = false;
    if (s < e && (*s == '+' || *s == '-')) neg = *s++ == '-';
    if (s == e || e - s > 18) return 1;
    long long v = 0;
    for (; s < e; ++s) {
        if (!mm_digit(*s)) return 1;
        v = v * 10 + (*s - '0');
    }
    out = neg ? -v : v;
    return 0;
}

#include "sgap_pow5.inc"

// Eisel-Lemire (Lemire, "Number Parsing at a Gigabyte per Second", 2021):
// w * 10^q correctly rounded to binary64 for w < 2^64 from the 128-bit
// truncated 5^q (sgap_pow5.inc), one 64x64 product plus a second one when
// the first leaves the rounding undecided.  Returns false (the host converts
// the token) where the method cannot decide or the result is not a normal
// finite double: |q| outside the table, a still-ambiguous product outside
// q in [-27, 55], subnormal or overflowing results.
__device__ __forceinline__ bool mm_eisel_lemire(unsigned long long w, int q, double &out) {
    if (q < SGAP_POW5_MIN_Q || q > SGAP_POW5_MAX_Q) return false;
    const int lz = __clzll((long long)w);
    w <<= lz;
    const unsigned long long *t = kPow5 + 2 * (q - SGAP_POW5_MIN_Q);
    unsigned long long hi = __umul64hi(w, t[0]);
    unsigned long long lo = w * t[0];
    if ((hi & 0x1FFULL) == 0x1FFULL) {
        const unsigned long long sh = __umul64hi(w, t[1]);
        lo += sh;
        if (sh > lo) ++hi;
        if (lo == ~0ULL && (q < -27 || q > 55)) return false;
    }
    const int upper = (int)(hi >> 63);
    const int shift = upper + 9;
    unsigned long long mant = hi >> shift;
    // floor(log2(10^q)) + 63 as (217706 q) >> 16, arithmetic shift
    long long p2 = ((217706LL * q) >> 16) + 63 + upper - lz + 1023;
    if (p2 <= 0) return false;
    if (lo <= 1 && q >= -4 && q <= 23 && (mant & 3) == 1 && (mant << shift) == hi)
        mant &= ~1ULL;  // exactly halfway: round to even
    mant += mant & 1;
    mant >>= 1;
    if (mant >= (2ULL << 52)) {
        mant = 1ULL << 52;
        ++p2;
    }
    mant &= ~(1ULL << 52);
    if (p2 >= 2047) return false;
    out = __longlong_as_double((long long)(((unsigned long long)p2 << 52) | mant));
    return true;
}

// Strict decimal float, correctly rounded: Clinger's fast path (mantissa
// <= 2^53, |decimal exponent| <= 22: one IEEE multiply or divide of two
// exact doubles) and Eisel-Lemire for the rest of <= 19 significant digits.
// 0 ok; 1 plain decimal neither method takes (> 19 significant digits,
// subnormal/overflowing, undecided: the host converts it); 2 anything else
// (inf/nan/underscores/...: Python judges the whole line).
__device__ __forceinline__ int mm_float(const unsigned char *s, const unsigned char *e, double &out) {
    const double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                            1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
    bool neg = false;
    if (s < e && (*s == '+' || *s == '-')) neg = *s++ == '-';
    unsigned long long w = 0;
    int sig = 0, frac = 0, nd = 0;
    bool hard = false;  // more than 19 significant digits
    for (; s < e && mm_digit(*s); ++s, ++nd) {
        if (w == 0 && *s == '0') continue;
        if (++sig > 19) hard = true; else w = w * 10 + (unsigned long long)(*s - '0');
    }
    if (s < e && *s == '.') {
        ++s;
        for (; s < e && mm_digit(*s); ++s, ++nd) {
            ++frac;
            if (w == 0 && *s == '0') continue;
            if (++sig > 19) hard = true; else w = w * 10 + (unsigned long long)(*s - '0');
        }
    }
    if (nd == 0) return 2;
    int ex = 0;
    if (s < e && (*s == 'e' || *s == 'E')) {
        ++s;
        bool eneg = false;
        if (s < e && (*s == '+' || *s == '-')) eneg = *s++ == '-';
        if (s == e) return 2;
        for (; s < e; ++s) {
            if (!mm_digit(*s)) return 2;
            if (ex < 100000) ex = ex * 10 + (*s - '0');
        }
        if (eneg) ex = -ex;
    }
    if (s != e) return 2;
    if (hard) return 1;
    const int d = ex - frac;
    double v;
    if (w == 0) {
        v = 0.0;
    } else {
        if (w <= (1ULL << 53) && d >= -22 && d <= 22)
            v = d >= 0 ? __dmul_rn((double)w, p10[d]) : __ddiv_rn((double)w, p10[-d]);
        else if (!mm_eisel_lemire(w, d, v))
            return 1;
    }
    out = neg ? -v : v;
    return 0;
}

// One thread per line: status + (row-1, col-1, value) for entries.
__global__ void k_mm_parse(const unsigned char *__restrict__ t, long long len,
                           const long long *__restrict__ starts, long long nlines, long long rows,
                           long long cols, unsigned char *__restrict__ status,
                           long long *__restrict__ r_out, long long *__restrict__ c_out,
                           double *__restrict__ v_out, long long *__restrict__ tok_off,
                           int *__restrict__ tok_len) {
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < nlines;
         l += (long long)gridDim.x * blockDim.x) {
        const unsigned char *p = t + starts[l];
        // at the line's '\n' (the last line may end at EOF or at a final '\n')
        const unsigned char *end =
            t + (l + 1 < nlines ? starts[l + 1] - 1 : (t[len - 1] == '\n' ? len - 1 : len));
        while (p < end && mm_space(*p)) ++p;
        if (p == end || *p == '%') {
            status[l] = kMmSkip;
            continue;
        }
        const unsigned char *tb[3], *te[3];
        int ntok = 0;
        while (p < end) {
            const unsigned char *q = p;
            while (q < end && !mm_space(*q)) ++q;
            if (ntok < 3) {
                tb[ntok] = p;
                te[ntok] = q;
            }
            ++ntok;
            p = q;
            while (p < end && mm_space(*p)) ++p;
        }
        if (ntok != 3) {
            status[l] = kMmFields;
            continue;
        }
        long long r, c;
        double v = 0.0;
        if (mm_int(tb[0], te[0], r) || mm_int(tb[1], te[1], c)) {
            status[l] = kMmHost;  // Python decides: exotic but valid, or non-numeric
            continue;
        }
        const int fv = mm_float(tb[2], te[2], v);
        if (fv == 2) {
            status[l] = kMmHost;
            continue;
        }
        if (r < 1 || r > rows || c < 1 || c > cols) {
            status[l] = kMmRange;
            continue;
        }
        status[l] = fv == 0 ? kMmOk : kMmFloat;
        tok_off[l] = tb[2] - t;
        tok_len[l] = (int)(te[2] - tb[2]);
        r_out[l] = r - 1;
        c_out[l] = c - 1;
        v_out[l] = v;
    }
}

// COO expansion in the reference's append order (matrices.py:195-200): each
// entry at pos[l], its symmetric mirror (off-diagonal) right after it.
// Keys are (row << 32 | col) so a stable sort reproduces np.lexsort.
__global__ void k_mm_expand(long long nlines, const unsigned char *__restrict__ status,
                            const long long *__restrict__ r, const long long *__restrict__ c,
                            const double *__restrict__ v, const long long *__restrict__ pos,
                            int symmetric, long long *__restrict__ key, double *__restrict__ val) {
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < nlines;
         l += (long long)gridDim.x * blockDim.x) {
        if (status[l] != kMmOk) continue;
        const long long o = pos[l];
        key[o] = (r[l] << 32) | c[l];
        val[o] = v[l];
        if (symmetric && r[l] != c[l]) {
            key[o + 1] = (c[l] << 32) | r[l];
            val[o + 1] = v[l];
        }
    }
}

// numpy's pairwise_sum (loops_utils.h): < 8 terms sequential from -0.0, <= 128
// eight interleaved accumulators, larger halves split at a multiple of 8.
__device__ double np_pairwise(const double *a, long long n) {
    // iterative over the recursion: a small explicit stack of (offset, n)
    struct Frame { long long off, n; double left; int state; };
    Frame st[40];
    int sp = 0;
    st[0] = {0, n, 0.0, 0};
    double ret = 0.0;
    while (sp >= 0) {
        Frame &f = st[sp];
        if (f.n <= 128) {
            double res;
            const double *x = a + f.off;
            if (f.n < 8) {
                res = -0.0;  // numpy starts from -0.0 (a sum of negative zeros stays -0.0)
                for (long long i = 0; i < f.n; ++i) res = __dadd_rn(res, x[i]);
            } else {
                double r8[8];
                for (int j = 0; j < 8; ++j) r8[j] = x[j];
                long long i = 8;
                for (; i < f.n - (f.n % 8); i += 8)
                    for (int j = 0; j < 8; ++j) r8[j] = __dadd_rn(r8[j], x[i + j]);
                res = __dadd_rn(__dadd_rn(__dadd_rn(r8[0], r8[1]), __dadd_rn(r8[2], r8[3])),
                                __dadd_rn(__dadd_rn(r8[4], r8[5]), __dadd_rn(r8[6], r8[7])));
                for (; i < f.n; ++i) res = __dadd_rn(res, x[i]);
            }
            ret = res;
            --sp;
            continue;
        }
        long long n2 = f.n / 2;
        n2 -= n2 % 8;
        if (f.state == 0) {  // descend left
            f.state = 1;
            st[++sp] = {f.off, n2, 0.0, 0};
        } else if (f.state == 1) {  // left done: descend right
            f.left = ret;
            f.state = 2;
            st[++sp] = {f.off + n2, f.n - n2, 0.0, 0};
        } else {  // both done
            ret = __dadd_rn(f.left, ret);
            --sp;
        }
    }
    return ret;
}

// One thread per run of equal keys in the sorted COO: np.add.reduceat order,
// i.e. a[s] + pairwise_sum(a[s+1:e]) (checked against numpy in the tests).
__global__ void k_mm_sum_runs(long long total, const long long *__restrict__ key,
                              const double *__restrict__ val, const long long *__restrict__ run_start,
                              long long nruns, long long *__restrict__ row, long long *__restrict__ col,
                              double *__restrict__ out) {
    for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < nruns;
         u += (long long)gridDim.x * blockDim.x) {
        const long long s = run_start[u];
        const long long e = u + 1 < nruns ? run_start[u + 1] : total;
        const double sum = e - s > 1 ? __dadd_rn(val[s], np_pairwise(val + s + 1, e - s - 1)) : val[s];
        const long long k = key[s];
        row[u] = k >> 32;
        col[u] = k & 0xffffffffLL;
        out[u] = sum;
    }
}

// row_ptr[r] = first position of row >= r in the sorted rows (a lower bound
// per row: the same integers as the reference's np.add.at + cumsum).
__global__ void k_mm_row_ptr(const long long *__restrict__ row, long long nnz, long long num_rows,
                             long long *__restrict__ row_ptr) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r <= num_rows;
         r += (long long)gridDim.x * blockDim.x) {
        long long lo = 0, hi = nnz;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (row[mid] < r) lo = mid + 1; else hi = mid;
        }
        row_ptr[r] = lo;
    }
}

}  // namespace sgap
