// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points onto the UNMODIFIED reference `warplm` field/io
// code (compiled from /root/reference/proj/src/*.cpp where it lies, by
// oracle/Makefile, into oracle/_ref/).  Used to pin the oracle's restatement
// bit-for-bit and to generate tests/golden fixtures.  Exceptions are mapped
// to status codes / NaN so they never cross the C boundary.
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

#include "warplm/field.hpp"
#include "warplm/io.hpp"

namespace {
warplm::Dims3 dims(int nx, int ny, int nz) {
    warplm::Dims3 d;
    d.nx = nx; d.ny = ny; d.nz = nz;
    return d;
}
warplm::Volume3 vol(const double* p, int nx, int ny, int nz) {
    warplm::Volume3 v(dims(nx, ny, nz));
    std::memcpy(v.data.data(), p, sizeof(double) * v.data.size());
    return v;
}
warplm::DispField3 fld(const double* p, int nx, int ny, int nz) {
    warplm::DispField3 f(dims(nx, ny, nz));
    std::memcpy(f.data.data(), p, sizeof(double) * f.data.size());
    return f;
}
constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
}  // namespace

extern "C" {

double ref_sample_trilinear_grad(const double* v, int nx, int ny, int nz, double px,
                                 double py, double pz, double* grad3) {
    const warplm::SampleGrad s = warplm::sample_trilinear_grad(vol(v, nx, ny, nz), px, py, pz);
    if (grad3) { grad3[0] = s.grad[0]; grad3[1] = s.grad[1]; grad3[2] = s.grad[2]; }
    return s.value;
}

// Whole-volume warp via per-voxel reference sample_trilinear_grad.
void ref_warp_volume(const double* M, const double* u, int nx, int ny, int nz, double* Mw,
                     double* gradM) {
    const warplm::Volume3 m = vol(M, nx, ny, nz);
    size_t i = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x, ++i) {
                const warplm::SampleGrad s = warplm::sample_trilinear_grad(
                    m, x + u[3 * i], y + u[3 * i + 1], z + u[3 * i + 2]);
                Mw[i] = s.value;
                if (gradM) for (int c = 0; c < 3; ++c) gradM[3 * i + c] = s.grad[c];
            }
}

void ref_sample_field(const double* u, int nx, int ny, int nz, double px, double py,
                      double pz, double* out3) {
    const warplm::Vec3 r = warplm::sample_field(fld(u, nx, ny, nz), px, py, pz);
    out3[0] = r[0]; out3[1] = r[1]; out3[2] = r[2];
}

int ref_compose_warp(const double* u, int nx, int ny, int nz, const double* v, int vnx,
                     int vny, int vnz, double eps, double* out) {
    try {
        const warplm::DispField3 r =
            warplm::compose_warp(fld(u, nx, ny, nz), fld(v, vnx, vny, vnz), eps);
        std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return 2;
    }
}

double ref_max_abs_component(const double* v, int nx, int ny, int nz) {
    return warplm::max_abs_component(fld(v, nx, ny, nz));
}

double ref_normalize_step(const double* v, int nx, int ny, int nz, double target, double fl) {
    warplm::StepScale s;
    s.target_max_disp = target;
    s.floor = fl;
    try {
        return warplm::normalize_step(fld(v, nx, ny, nz), s);
    } catch (const std::invalid_argument&) {
        return kNaN;
    }
}

double ref_jacobian_det_min(const double* u, int nx, int ny, int nz) {
    try {
        return warplm::jacobian_det_min(fld(u, nx, ny, nz));
    } catch (const std::invalid_argument&) {
        return kNaN;
    }
}

void ref_gaussian_smooth(double* data, int nx, int ny, int nz, int nchan, double sigma) {
    if (nchan == 1) {
        const warplm::Volume3 r = warplm::gaussian_smooth(vol(data, nx, ny, nz), sigma);
        std::memcpy(data, r.data.data(), sizeof(double) * r.data.size());
    } else {
        const warplm::DispField3 r = warplm::gaussian_smooth(fld(data, nx, ny, nz), sigma);
        std::memcpy(data, r.data.data(), sizeof(double) * r.data.size());
    }
}

int ref_all_finite(const double* data, int nx, int ny, int nz, int nchan) {
    return nchan == 1 ? warplm::all_finite(vol(data, nx, ny, nz))
                      : warplm::all_finite(fld(data, nx, ny, nz));
}

// io.cpp round trips.  Return 0 ok, 1 io_error (message copied to err).
int ref_write_vol3(const char* path, const double* data, int nx, int ny, int nz, char* err,
                   int errlen) {
    try {
        warplm::write_vol3(path, vol(data, nx, ny, nz));
        return 0;
    } catch (const warplm::io_error& e) {
        if (err && errlen > 0) { std::strncpy(err, e.what(), errlen - 1); err[errlen - 1] = 0; }
        return 1;
    }
}
int ref_write_dsp3(const char* path, const double* data, int nx, int ny, int nz, char* err,
                   int errlen) {
    try {
        warplm::write_dsp3(path, fld(data, nx, ny, nz));
        return 0;
    } catch (const warplm::io_error& e) {
        if (err && errlen > 0) { std::strncpy(err, e.what(), errlen - 1); err[errlen - 1] = 0; }
        return 1;
    }
}
// Reads header + payload; dims3 receives (nx, ny, nz); data may be null to
// query dims only (payload still validated).
int ref_read(const char* path, int is_field, int* dims3, double* data, size_t cap, char* err,
             int errlen) {
    try {
        if (is_field) {
            const warplm::DispField3 f = warplm::read_dsp3(path);
            dims3[0] = f.dims.nx; dims3[1] = f.dims.ny; dims3[2] = f.dims.nz;
            if (data && cap >= f.data.size()) std::memcpy(data, f.data.data(), sizeof(double) * f.data.size());
        } else {
            const warplm::Volume3 v = warplm::read_vol3(path);
            dims3[0] = v.dims.nx; dims3[1] = v.dims.ny; dims3[2] = v.dims.nz;
            if (data && cap >= v.data.size()) std::memcpy(data, v.data.data(), sizeof(double) * v.data.size());
        }
        return 0;
    } catch (const warplm::io_error& e) {
        if (err && errlen > 0) { std::strncpy(err, e.what(), errlen - 1); err[errlen - 1] = 0; }
        return 1;
    }
}

}  // extern "C"
