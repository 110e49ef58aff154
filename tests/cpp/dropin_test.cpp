// Drop-in check: code written against the reference API builds both the
// reference igabem::H2Matrix (oracle/_ref) and igabem_b200::H2Matrix (B200)
// from the same igabem::Discretization and compares them.  Needs a GPU.
#include <cstdio>
#include <memory>
#include <random>

#include <igabem/h2.hpp>
#include <igabem/shapes.hpp>
#include <igabem_b200/h2_dropin.hpp>

using namespace igabem;

template <typename Scalar>
double run(const Discretization& d, H2Options o) {
  H2Matrix<Scalar> ref(d, o);
  igabem_b200::H2Matrix<Scalar> b200(d, o);
  if (ref.nearfield_pairs() != b200.nearfield_pairs() || ref.farfield_pairs() != b200.farfield_pairs()) return 1.0;
  const auto s1 = ref.storage_report(), s2 = b200.storage_report();
  if (s1.total_bytes != s2.total_bytes || s1.nearfield_entries != s2.nearfield_entries) return 1.0;
  std::mt19937_64 rng(20261019);
  std::uniform_real_distribution<double> u(-1, 1);
  Eigen::Matrix<Scalar, Eigen::Dynamic, 1> x(d.dof_count());
  for (int i = 0; i < x.size(); ++i) {
    if constexpr (std::is_same_v<Scalar, double>) x[i] = u(rng);
    else x[i] = Scalar(u(rng), u(rng));
  }
  const auto y1 = ref * x;
  const auto y2 = b200 * x;
  return (y1 - y2).norm() / y1.norm();
}

int main() {
  auto sphere = std::make_shared<const Geometry>(make_sphere());
  int fails = 0;
  {
    Discretization d(sphere, Pde::laplace(), 2, 1, 3);
    const double e = run<double>(d, {.m = 8, .eta = 1.6});
    std::printf("laplace P2 L3 m8: rel %.3e\n", e);
    fails += !(e < 1e-10);
  }
  {
    Discretization d(sphere, Pde::helmholtz(cplx(3, 0)), 1, 1, 2);
    const double e = run<cplx>(d, {.m = 6, .eta = 1.6});
    std::printf("helmholtz P1 L2 m6: rel %.3e\n", e);
    fails += !(e < 1e-10);
  }
  {
    Discretization d(sphere, Pde::maxwell(cplx(2 * M_PI, 0)), 2, 1, 2);
    const double e = run<cplx>(d, {.m = 6, .eta = 1.6});
    std::printf("maxwell P2 L2 m6: rel %.3e\n", e);
    fails += !(e < 1e-10);
  }
  try {
    Discretization d(sphere, Pde::laplace(), 1, 1, 1);
    igabem_b200::H2Matrix<cplx> bad(d);
    ++fails;
  } catch (const std::invalid_argument&) {
  }
  std::printf(fails ? "FAIL\n" : "OK\n");
  return fails;
}
