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
    if (sb > 1e-12) {
        e.a = atan2(m12, m02);
        e.g = atan2(m21, -m20);
    } else if (m22 > 0.0) {
        e.a = atan2(m10, m00);
        e.g = 0.0;
    } else {
        e.a = atan2(-m10, -m00);
        e.g = 0.0;
    }
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
    double a[3][3];
    int rp[3], cp[3];
    int nz;
    double maxpiv;
    BMB_HD void factor(const double m[9]) {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) a[i][j] = m[i * 3 + j];
        nz = 3;
        maxpiv = 0.0;
        for (int k = 0; k < 3; ++k) {
            int br = k, bc = k;
            double big = -1.0;
            for (int j = k; j < 3; ++j)
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
                for (int i = k; i < 3; ++i) rp[i] = cp[i] = i;
                break;
            }
            if (big > maxpiv) maxpiv = big;
            rp[k] = br;
            cp[k] = bc;
            if (br != k)
                for (int j = 0; j < 3; ++j) {
                    const double t = a[k][j];
                    a[k][j] = a[br][j];
                    a[br][j] = t;
                }
            if (bc != k)
                for (int i = 0; i < 3; ++i) {
                    const double t = a[i][k];
                    a[i][k] = a[i][bc];
                    a[i][bc] = t;
                }
            if (k < 2) {
                for (int i = k + 1; i < 3; ++i) a[i][k] /= a[k][k];
                for (int i = k + 1; i < 3; ++i)
                    for (int j = k + 1; j < 3; ++j) a[i][j] -= a[i][k] * a[k][j];
            }
        }
    }
    BMB_HD bool invertible() const {
        const double thr = 2.220446049250313e-16 * 3.0 * fabs(maxpiv);
        int rank = 0;
        for (int i = 0; i < nz; ++i)
            if (fabs(a[i][i]) > thr) ++rank;
        return rank == 3;
    }
    BMB_HD void solve(const double b[3], double x[3]) const {
        double c[3] = {b[0], b[1], b[2]};
        for (int k = 0; k < 3; ++k)
            if (rp[k] != k) {
                const double t = c[k];
                c[k] = c[rp[k]];
                c[rp[k]] = t;
            }
        for (int i = 1; i < 3; ++i)
            for (int j = 0; j < i; ++j) c[i] -= a[i][j] * c[j];
        for (int i = 2; i >= 0; --i) {
            for (int j = i + 1; j < 3; ++j) c[i] -= a[i][j] * c[j];
            c[i] /= a[i][i];
        }
        for (int k = 2; k >= 0; --k)
            if (cp[k] != k) {
                const double t = c[k];
                c[k] = c[cp[k]];
                c[cp[k]] = t;
            }
        x[0] = c[0];
        x[1] = c[1];
        x[2] = c[2];
    }
};

}  // namespace bmb
