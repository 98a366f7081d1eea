// FP64 rotation helpers usable on host and device: unit quaternions (w,x,y,z),
// active rotations, ZYZ Euler view.  Same conventions as the reference's
// Rotation (include/ballmatch/rotation.hpp:16-50, src/rotation.cpp).
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define BMB_HD __host__ __device__ __forceinline__
#else
#define BMB_HD inline
#endif

namespace bmb {

struct Quat {
    double w, x, y, z;
};
struct Euler3 {
    double a, b, g;
};

BMB_HD Quat q_normalized(double w, double x, double y, double z) {
    const double n = sqrt(w * w + x * x + y * y + z * z);
    return {w / n, x / n, y / n, z / n};
}
// product a*b: b applied first (rotation.cpp:95-100, unnormalized)
BMB_HD Quat q_mul(const Quat& a, const Quat& b) {
    return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
            a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
            a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
            a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
BMB_HD Quat q_inv(const Quat& a) { return {a.w, -a.x, -a.y, -a.z}; }
// rotation about a unit coordinate axis (from_axis_angle, rotation.cpp:23-29)
BMB_HD Quat q_axis(int axis, double angle) {
    const double h = 0.5 * angle, s = sin(h);
    return q_normalized(cos(h), axis == 0 ? s : 0.0, axis == 1 ? s : 0.0, axis == 2 ? s : 0.0);
}
// Rz(a) Ry(b) Rz(g) (rotation.cpp:31-34)
BMB_HD Quat q_from_euler(double a, double b, double g) {
    return q_mul(q_mul(q_axis(2, a), q_axis(1, b)), q_axis(2, g));
}
// ZYZ angles with beta in [0, pi] and the pole conventions of rotation.cpp:77-93
BMB_HD Euler3 q_euler(const Quat& q) {
    const double w = q.w, x = q.x, y = q.y, z = q.z;
    const double m00 = 1 - 2 * (y * y + z * z), m02 = 2 * (x * z + w * y);
    const double m10 = 2 * (x * y + w * z), m12 = 2 * (y * z - w * x);
    const double m20 = 2 * (x * z - w * y), m21 = 2 * (y * z + w * x);
    const double m22 = 1 - 2 * (x * x + y * y);
    Euler3 e;
    const double sb = hypot(m02, m12);
    e.b = atan2(sb, m22);
    // one atan2 per angle (the branches pick its arguments; atan2(0, 1) = +0)
    double ya = m12, xa = m02, yg = m21, xg = -m20;
    if (!(sb > 1e-12)) {
        const double s = m22 > 0.0 ? 1.0 : -1.0;
        ya = s * m10, xa = s * m00, yg = 0.0, xg = 1.0;
    }
    e.a = atan2(ya, xa);
    e.g = atan2(yg, xg);
    return e;
}
// geodesic angle to the identity, radians (angle_to, rotation.cpp:102-107)
BMB_HD double q_angle(const Quat& q) {
    const double v = sqrt(q.x * q.x + q.y * q.y + q.z * q.z);
    return 2.0 * atan2(v, fabs(q.w));
}

// Eigen::FullPivLU<Matrix3d> semantics for the damped Newton step
// (src/optimize.cpp:316-323): full pivoting in column-major search order,
// rank threshold = eps * 3 * |largest pivot|.
struct LU3 {
    // every index below is a compile-time constant after unrolling (the pivot
    // swaps are predicated), so the factors stay in registers
    double a[3][3];
    int rp[3], cp[3];
    int nz;
    double maxpiv;
    static BMB_HD void swap_(double& x, double& y) {
        const double t = x;
        x = y;
        y = t;
    }
    BMB_HD void factor(const double m[9]) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) a[i][j] = m[i * 3 + j];
        nz = 3;
        maxpiv = 0.0;
        bool stop = false;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (stop) {
                rp[k] = cp[k] = k;
                continue;
            }
            int br = k, bc = k;
            double big = -1.0;
#pragma unroll
            for (int j = k; j < 3; ++j)
#pragma unroll
                for (int i = k; i < 3; ++i) {
                    const double v = fabs(a[i][j]);
                    if (v > big) {
                        big = v;
                        br = i;
                        bc = j;
                    }
                }
            if (big == 0.0) {
                nz = k;
                stop = true;
                rp[k] = cp[k] = k;
                continue;
            }
            if (big > maxpiv) maxpiv = big;
            rp[k] = br;
            cp[k] = bc;
#pragma unroll
            for (int i = k + 1; i < 3; ++i)
                if (br == i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) swap_(a[k][j], a[i][j]);
#pragma unroll
            for (int j = k + 1; j < 3; ++j)
                if (bc == j)
#pragma unroll
                    for (int i = 0; i < 3; ++i) swap_(a[i][k], a[i][j]);
            if (k < 2) {
#pragma unroll
                for (int i = k + 1; i < 3; ++i) a[i][k] /= a[k][k];
#pragma unroll
                for (int i = k + 1; i < 3; ++i)
#pragma unroll
                    for (int j = k + 1; j < 3; ++j) a[i][j] -= a[i][k] * a[k][j];
            }
        }
    }
    BMB_HD bool invertible() const {
        const double thr = 2.220446049250313e-16 * 3.0 * fabs(maxpiv);
        int rank = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            if (i < nz && fabs(a[i][i]) > thr) ++rank;
        return rank == 3;
    }
    BMB_HD void solve(const double b[3], double x[3]) const {
        // P^T b (rows), L and U substitutions, then Q (columns) -- written out in
        // scalars so that nothing is addressed dynamically
        double c0 = b[0], c1 = b[1], c2 = b[2], t;
        if (rp[0] == 1) t = c0, c0 = c1, c1 = t;
        else if (rp[0] == 2) t = c0, c0 = c2, c2 = t;
        if (rp[1] == 2) t = c1, c1 = c2, c2 = t;
        c1 -= a[1][0] * c0;
        c2 -= a[2][0] * c0;
        c2 -= a[2][1] * c1;
        c2 /= a[2][2];
        c1 -= a[1][2] * c2;
        c1 /= a[1][1];
        c0 -= a[0][1] * c1;
        c0 -= a[0][2] * c2;
        c0 /= a[0][0];
        if (cp[1] == 2) t = c1, c1 = c2, c2 = t;
        if (cp[0] == 1) t = c0, c0 = c1, c1 = t;
        else if (cp[0] == 2) t = c0, c0 = c2, c2 = t;
        x[0] = c0;
        x[1] = c1;
        x[2] = c2;
    }
};

}  // namespace bmb
