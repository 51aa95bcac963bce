// abed/abft_gemm.hpp -- drop-in for the reference's abft_gemm.hpp: the classical
// row/column-checksum ABFT for an int8 GEMM that the paper contrasts with ABED.
//
// abft_gemm runs its online tasks on the B200 through libabed_b200.so (the GEMM on
// the tcgen05 kernel, the checksum row / column as base-256 digit rows, the dual
// output-checksum comparison as separate passes -- csrc/abft.cu); abft_check runs
// on the device too.  c, c_aug and both VerifyOutcomes are bit-identical to the
// reference (tests/test_gpu_abft.py).  abft_costs is the reference's task
// accounting (host arithmetic).
// citations: abft_gemm.hpp:17-39 AbftTaskCost / AbftCosts, :41-55 abft_costs,
// :57-65 AbftResult, :70-96 abft_check, :102-152 abft_gemm.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string_view>
#include <utility>

#include "checksum.hpp"
#include "convolution.hpp"
#include "device.hpp"

namespace abed {

/// One online ABFT task: (2) copy-in, (3) input checksums, (4) GEMM, (5) output
/// checksums + comparison, (6) copy-out.
struct AbftTaskCost {
  std::string_view name;
  std::int64_t ops = 0;
  std::int64_t read_bytes = 0;
  std::int64_t write_bytes = 0;
  std::int64_t elements_moved = 0;
};

struct AbftCosts {
  std::array<AbftTaskCost, 5> tasks;  // tasks (2) .. (6)

  std::int64_t copy_elements() const { return tasks[0].elements_moved + tasks[4].elements_moved; }
  std::int64_t total_ops() const {
    std::int64_t sum = 0;
    for (const auto& t : tasks) sum += t.ops;
    return sum;
  }
  std::int64_t total_bytes() const {
    std::int64_t sum = 0;
    for (const auto& t : tasks) sum += t.read_bytes + t.write_bytes;
    return sum;
  }
};

/// The reference's accounting: i8 operands widened to i32 augmented copies,
/// an (m+1) x (n+1) i64 product, one or two passes over it for the checks.
inline AbftCosts abft_costs(std::int64_t m, std::int64_t n, std::int64_t k, bool single_pass_output_check = false) {
  const std::int64_t in_elems = m * k + k * n;
  const std::int64_t aug = (m + 1) * (n + 1);
  AbftCosts c;
  c.tasks[0] = {"copy_in", 0, in_elems, in_elems * 4, in_elems};
  c.tasks[1] = {"input_checksums", k * (m - 1) + k * (n - 1), in_elems, 2 * k * 4, 0};
  c.tasks[2] = {"gemm", aug * k, ((m + 1) * k + k * (n + 1)) * 4, aug * 8, 0};
  c.tasks[3] = {"output_checksums", (m + 1) * (n - 1) + (n + 1) * (m - 1) + (m + 1) + (n + 1),
                (single_pass_output_check ? 1 : 2) * aug * 8, 8, 0};
  c.tasks[4] = {"copy_out", 0, m * n * 8, m * n * 4, 2 * m * n};
  return c;
}

struct AbftResult {
  Matrix c;                 // m x n, i32
  Matrix c_aug;             // (m+1) x (n+1), i64
  VerifyOutcome row_check;  // row sums vs the appended column
  VerifyOutcome col_check;  // column sums vs the appended row
  AbftCosts costs;

  bool pass() const { return row_check.pass() && col_check.pass(); }
};

/// Row check over rows 0..m, column check over columns 0..n; each reports its
/// first mismatch with locus (index, -1, -1).
inline std::pair<VerifyOutcome, VerifyOutcome> abft_check(const Matrix& c_aug) {
  if (c_aug.rows < 2 || c_aug.cols < 2) throw std::invalid_argument("abft_check: matrix too small");
  if (c_aug.kind != ElemKind::I64) throw std::invalid_argument("abft_check: c_aug must be i64");
  const device::Buffer d = device::upload(c_aug.data.data(), c_aug.data.size());
  abed_verify_outcome row{}, col{};
  device::check(abed_abft_check(d.get<int64_t>(), c_aug.rows, c_aug.cols, &row, &col));
  return {detail::from_c(row), detail::from_c(col)};
}

/// Row/column-checksum ABFT for an int8 GEMM (detection only).
inline AbftResult abft_gemm(const Matrix& a, const Matrix& b, bool single_pass_output_check = false) {
  if (a.kind != ElemKind::I8 || b.kind != ElemKind::I8) throw std::invalid_argument("abft_gemm: operands must be i8");
  if (a.cols != b.rows) throw std::invalid_argument("abft_gemm: inner dimensions do not match");
  const std::int64_t m = a.rows, k = a.cols, n = b.cols;
  const device::Buffer da = device::upload(a.data.data(), a.data.size());
  const device::Buffer db = device::upload(b.data.data(), b.data.size());
  device::Buffer dc(static_cast<std::size_t>(m * n) * 4), dca(static_cast<std::size_t>((m + 1) * (n + 1)) * 8);
  abed_verify_outcome row{}, col{};
  device::check(abed_abft_gemm_i8(da.get<int8_t>(), m, k, db.get<int8_t>(), b.rows, n, dc.get<int32_t>(),
                                  dca.get<int64_t>(), &row, &col));
  AbftResult r;
  r.c = Matrix(m, n, ElemKind::I32);
  r.c_aug = Matrix(m + 1, n + 1, ElemKind::I64);
  device::download(dc, r.c.data.data(), r.c.data.size());
  device::download(dca, r.c_aug.data.data(), r.c_aug.data.size());
  r.row_check = detail::from_c(row);
  r.col_check = detail::from_c(col);
  r.costs = abft_costs(m, n, k, single_pass_output_check);
  return r;
}

}  // namespace abed
