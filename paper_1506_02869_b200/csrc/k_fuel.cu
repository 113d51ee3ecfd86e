// k_fuel.cu -- the two fuel estimates of section 5 on batches of
// recorded traces: one thread per aircraft trace, sequential over its samples
// (the mass recursion), FP64.  Off the MPC hot path; written from the paper's
// equations (reading R47 for the silent points).
#include <cmath>

#include "../../include/smcatm.h"
#include "smc_device.cuh"

namespace smc {

__device__ __forceinline__ double fuel_density(int mode, double rho_const, double z) {
    if (mode != 0) return rho_const;
    const double base = 1.0 - 2.2558e-5 * z;
    return 1.225 * pow(base > 0.0 ? base : 0.0, 4.2559);
}

// parabolic polar, coordinated-turn lift C_L = m g / (q cos phi) (R12)
__device__ __forceinline__ double fuel_drag(const smc_fuel_type &a, int mode, double rho_const, double g, double z,
                                            double v, double m, double phi) {
    const double qd = 0.5 * fuel_density(mode, rho_const, z) * v * v * a.S;
    const double CL = m * g / cos(phi) / qd;
    return qd * (a.cd0 + a.cd2 * CL * CL);
}

// gamma = asin(dz / (dt v)); outside [-1, 1] (degenerate data) -> +-gamma_max, flagged (R47)
__device__ __forceinline__ double fuel_gamma(double sg, double gmax, uint32_t &flags) {
    if (!(sg >= -1.0 && sg <= 1.0)) { flags |= 1u; return sg > 0.0 ? gmax : -gmax; }
    return asin(sg);
}

__global__ void k_fuel(const smc_fuel_args a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n_traces) return;
    const smc_fuel_type ty = a.type[i];
    const uint32_t K = a.len[i];
    const double *tr = a.trace + (size_t)i * a.max_len * 5;
    double *m1 = a.m1 + (size_t)i * a.max_len, *m2 = a.m2 + (size_t)i * a.max_len;
    double *w = a.wres + (size_t)i * a.max_len * 2;
    const double dt = a.dt, g = a.g;
    uint32_t flags = 0;
    double ma = a.m0[i], mb = a.m0[i];
    if (K > 0) { m1[0] = ma; m2[0] = mb; }
    for (uint32_t k = 0; k + 1 < K; ++k) {
        const double *p = tr + 5 * k, *q = tr + 5 * (k + 1);
        // ---- estimate 1: recorded heading and airspeed, wind as residual
        {
            const double vs = p[3];
            const double eta = ty.Cf1 * (1.0 + vs / ty.Cf2);
            const double gam = fuel_gamma((q[2] - p[2]) / (dt * vs), ty.gamma_max, flags);
            w[2 * k] = (q[0] - p[0]) / dt - vs * cos(p[4]) * cos(gam);
            w[2 * k + 1] = (q[1] - p[1]) / dt - vs * sin(p[4]) * cos(gam);
            const double D = fuel_drag(ty, a.density_mode, a.rho_const, g, p[2], vs, ma, 0.0);
            const double T = ma * (q[3] - vs) / dt + D + ma * g * sin(gam);
            const double burn = dt * eta * T;
            ma -= burn > 0.0 ? burn : 0.0;
            m1[k + 1] = ma;
        }
        // ---- estimate 2: dead reckoning, no wind
        {
            const double dx = q[0] - p[0], dy = q[1] - p[1], dz = q[2] - p[2];
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            if (!(d > 0.0)) {
                flags |= 2u;
            } else {
                const double vh = d / dt;
                const double eta = ty.Cf1 * (1.0 + vh / ty.Cf2);
                const double gam = fuel_gamma(dz / (dt * vh), ty.gamma_max, flags);
                const double chih = atan2(dy, dx);
                double dchi = chih - p[4];
                dchi -= 6.283185307179586 * floor((dchi + 3.141592653589793) / 6.283185307179586);
                const double phi = atan(dchi * vh / (g * dt));
                const double D = fuel_drag(ty, a.density_mode, a.rho_const, g, p[2], vh, mb, phi);
                const double T = mb * (q[3] - vh) / dt + D + mb * g * sin(gam);
                const double burn = dt * eta * T;
                mb -= burn > 0.0 ? burn : 0.0;
            }
            m2[k + 1] = mb;
        }
    }
    if (K > 0) { w[2 * (K - 1)] = 0.0; w[2 * (K - 1) + 1] = 0.0; }
    a.fuel[2 * i] = a.m0[i] - ma;
    a.fuel[2 * i + 1] = a.m0[i] - mb;
    a.flags[i] = flags;
}

}  // namespace smc

extern "C" smc_status smc_fuel_estimates(const smc_fuel_args *args, void *stream) {
    if (!args || !args->len || !args->trace || !args->m0 || !args->type || !args->m1 || !args->m2 || !args->wres ||
        !args->fuel || !args->flags || args->n_traces == 0 || args->max_len == 0 || !(args->dt > 0.0))
        return SMC_EINVAL;
    const unsigned blocks = (args->n_traces + 127) / 128;
    smc::k_fuel<<<blocks, 128, 0, (cudaStream_t)stream>>>(*args);
    return cudaGetLastError() == cudaSuccess ? SMC_OK : SMC_ECUDA;
}
