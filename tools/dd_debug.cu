// Debug harness: CUDA vs refined (double-double) acos/atan2 on bin-edge inputs.
#include <cstdio>
#include "../paper_2008_06972_b200/csrc/dd.cuh"
using namespace stpc;
__global__ void k(const double* in, double* out, int n)
{
    int i = threadIdx.x;
    if (i >= n) return;
    double cz = in[2 * i], y = in[2 * i + 1];
    out[6 * i + 0] = acos(cz);
    out[6 * i + 1] = dd::acos_cr(cz);
    out[6 * i + 2] = atan2(cz, y);
    out[6 * i + 3] = dd::atan2_cr(cz, y);
    dd::D2 s, c;
    dd::sincos_dd(dd::D2{acos(cz), 0.0}, s, c);
    out[6 * i + 4] = s.hi;
    out[6 * i + 5] = s.lo;
}
int main()
{
    double h_in[8] = {0.70710678118654757, 1.0, 0.3, 0.7, -0.2, 2.0, 1e-3, -5.0};
    double *d_in, *d_out, h_out[24];
    cudaMalloc(&d_in, sizeof h_in);
    cudaMalloc(&d_out, sizeof h_out);
    cudaMemcpy(d_in, h_in, sizeof h_in, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(d_in, d_out, 4);
    cudaMemcpy(h_out, d_out, sizeof h_out, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 4; ++i)
        printf("in %.17g %.17g | acos %.17g cr %.17g | atan2 %.17g cr %.17g | sin %.17g %.17g\n", h_in[2 * i],
               h_in[2 * i + 1], h_out[6 * i], h_out[6 * i + 1], h_out[6 * i + 2], h_out[6 * i + 3],
               h_out[6 * i + 4], h_out[6 * i + 5]);
    return 0;
}
