// stats.cu -- factor statistics of convolution layers: the producer in front of the EA update.
//
// The reference's network is an MLP: A_l = [a_{l-1}; 1] ((d_in+1) x n, with_ones_row, network.hpp:94-95), G_l = the
// back-propagated signal (d_out x n, network.hpp:134), and accumulate_factors updates each factor with M = X / sqrt(n)
// (network.hpp:155-165).  For a convolution (the VGG16_bn layers of BASELINE config 3) the same statistics are taken
// over every output location (KFC): the A matrix is the patch matrix (im2col) with a ones row, d = C_in*kh*kw + 1
// rows and n = B*H_out*W_out columns, and G is the output-gradient tensor with n = B*H_out*W_out columns.  Both
// kernels write the EA operand M = X * scale (scale = 1/sqrt(n)) directly, row-major d x n with pitch ld, so the
// batched EA consumes them without another pass.
#include "kernels.cuh"

namespace rkfac_b200 {

namespace {

// out[row][col], row = (c*kh + ky)*kw + kx (+ the ones row last), col = (b*Ho + oy)*Wo + ox: one thread per output
// element along a row, so stores are coalesced and loads walk the input row (stride sw).
__global__ void patches_kernel(ConvPatchDesc p) {
    const long long n = (long long)p.B * p.Ho * p.Wo;
    const int rows = p.C * p.kh * p.kw + (p.ones ? 1 : 0);
    const int row = blockIdx.y;
    if (row >= rows) return;
    float* o = p.out + (long long)row * p.ld;
    if (p.ones && row == rows - 1) {
        for (long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x; col < n;
             col += (long long)gridDim.x * blockDim.x)
            o[col] = p.scale;
        return;
    }
    const int kx = row % p.kw, ky = (row / p.kw) % p.kh, c = row / (p.kw * p.kh);
    const long long hw = (long long)p.Ho * p.Wo;
    for (long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x; col < n;
         col += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(col / hw);
        const int rem = (int)(col - b * hw);
        const int oy = rem / p.Wo, ox = rem - oy * p.Wo;
        const int iy = oy * p.sh - p.ph + ky * p.dh, ix = ox * p.sw - p.pw + kx * p.dw;
        float v = 0.f;
        if (iy >= 0 && iy < p.H && ix >= 0 && ix < p.W)
            v = p.x[(((long long)b * p.C + c) * p.H + iy) * p.W + ix];
        o[col] = v * p.scale;
    }
}

// out[co][b*HoWo + q] = scale * dy[b][co][q]
__global__ void grads_kernel(const float* __restrict__ dy, int B, int Co, long long hw, float scale,
                             float* __restrict__ out, long long ld) {
    const int co = blockIdx.y;
    const long long n = (long long)B * hw;
    for (long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x; col < n;
         col += (long long)gridDim.x * blockDim.x) {
        const long long b = col / hw, q = col - b * hw;
        out[(long long)co * ld + col] = scale * dy[(b * Co + co) * hw + q];
    }
}

}  // namespace

void launch_conv_patches(const ConvPatchDesc& p, cudaStream_t s) {
    const long long n = (long long)p.B * p.Ho * p.Wo;
    const int rows = p.C * p.kh * p.kw + (p.ones ? 1 : 0);
    if (n == 0 || rows == 0) return;
    const int bx = (int)std::min<long long>(ceil_div(n, 256), std::max<long long>(1, 4096 / rows + 1));
    RKFAC_REQUIRE(rows <= 65535, RKFAC_INVALID_ARGUMENT, "conv patches: too many rows");
    patches_kernel<<<dim3(bx, rows), 256, 0, s>>>(p);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_conv_grads(const float* dy, int B, int Co, long long hw, float scale, float* out, long long ld,
                       cudaStream_t s) {
    const long long n = (long long)B * hw;
    if (n == 0 || Co == 0) return;
    RKFAC_REQUIRE(Co <= 65535, RKFAC_INVALID_ARGUMENT, "conv grads: too many channels");
    const int bx = (int)std::min<long long>(ceil_div(n, 256), std::max<long long>(1, 4096 / Co + 1));
    grads_kernel<<<dim3(bx, Co), 256, 0, s>>>(dy, B, Co, hw, scale, out, ld);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
