// pc2.cu -- placeholder (filled in by the PC2 milestone)
#include "pot3d_internal.cuh"
namespace pot3d {
struct Pc2 { int dummy; };
int pc2_create(Pc2 **out, const Grid &, int, const int *, void *(*)(size_t, void *), void *) { *out = nullptr; return -1; }
int pc2_factor(Pc2 *, const Metrics &, cudaStream_t, double *) { return -1; }
int pc2_apply(Pc2 *, const Metrics &, Scalars *, const double *, double *, double *, int, double *, cudaStream_t, bool) { return -1; }
void pc2_destroy(Pc2 *, void (*)(void *, void *), void *) {}
size_t pc2_bytes(const Pc2 *) { return 0; }
int pc2_kernels_per_apply(const Pc2 *) { return 0; }
}
