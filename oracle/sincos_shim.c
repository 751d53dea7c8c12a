/* oracle/sincos_shim.c — TEST INFRASTRUCTURE (parity checker only).
 *
 * Replaces libm's sin/cos/sincos inside the oracle builds with the pinned
 * routine the CUDA kernels inline (paper_2110_06879_b200/csrc/ga_sincos.h).
 * The reference calls std::cos/std::sin at proj/src/kernels.cpp:30-31,
 * proj/src/netdata.cpp:37-38 and std::polar at proj/src/netdata.cpp:20; GCC
 * lowers those to `sincos`/`sin`/`cos`.  The symbols here are linked into the
 * oracle shared objects with hidden visibility, so the static linker binds
 * every such call inside the oracle to this file instead of glibc's IFUNC
 * (whose bits depend on the host CPU).
 *
 * Must be compiled with -ffp-contract=off -fno-builtin.
 */
#include "../paper_2110_06879_b200/csrc/ga_sincos.h"

#define GA_HIDDEN __attribute__((visibility("hidden")))

GA_HIDDEN void sincos(double x, double* s, double* c) { ga_sincos(x, s, c); }
GA_HIDDEN double sin(double x) { return ga_sin(x); }
GA_HIDDEN double cos(double x) { return ga_cos(x); }

/* Exported probe so tests can compare host bits with device bits. */
void ga_oracle_sincos(double x, double* s, double* c) { ga_sincos(x, s, c); }

/* Batched probe (parity tests compare millions of arguments). */
void ga_oracle_sincos_batch(long n, const double* x, double* s, double* c) {
    for (long i = 0; i < n; ++i) ga_sincos(x[i], &s[i], &c[i]);
}
