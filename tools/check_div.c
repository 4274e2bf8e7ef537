/* tools/check_div.c: Markstein-corrected division a*RN(1/b) + fma residual == a/b (bit-identical) on stress operands.
   gcc -O2 -ffp-contract=off -march=native -o check_div tools/check_div.c -lm && ./check_div 300000000 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 1234567ull;
static inline uint64_t nx(void){ s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main(int argc, char** argv) {
    long n = atol(argv[1]); long bad = 0;
    for (long i = 0; i < n; ++i) {
        /* divisor mantissa near all-ones / all-zeros patterns, numerator random double of moderate exponent */
        uint64_t mant;
        int k = nx() % 4;
        if (k == 0) mant = 0xFFFFFFFFFFFFFull - (nx() % 1024);
        else if (k == 1) mant = nx() % 1024;
        else if (k == 2) mant = 0x8000000000000ull + (nx() % 4096) - 2048;
        else mant = nx() & 0xFFFFFFFFFFFFFull;
        uint64_t e = 1023 - (nx() % 60);
        uint64_t bits = (e << 52) | mant | ((nx() & 1) << 63);
        double d; memcpy(&d, &bits, 8);
        uint64_t ab = ((uint64_t)(1023 - 20 + nx() % 34) << 52) | (nx() & 0xFFFFFFFFFFFFFull) | ((nx() & 1) << 63);
        double a; memcpy(&a, &ab, 8);
        double inv = 1.0 / d;
        double q = a * inv;
        double r = fma(-q, d, a);
        double q1 = fma(r, inv, q);
        double want = a / d;
        if (memcmp(&q1, &want, 8) != 0) { if (bad < 10) printf("a=%a d=%a want=%a got=%a\n", a, d, want, q1); ++bad; }
    }
    printf("%ld mismatches of %ld\n", bad, n);
}
