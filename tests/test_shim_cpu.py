"""CPU-side checks of the dfs:: drop-in C++ shim: every reference hot-path
declaration (curve.hpp, mask_builder.hpp, attention.hpp, scheduler.hpp under
/root/reference/proj/include/dfs) is exported by libdfs_b200.so, and the
headers compile standalone. No kernel runs here."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_23445_b200", "libdfs_b200.so")

EXPECTED = [
    "dfs::ordering_name(", "dfs::parse_ordering(", "dfs::validate_permutation(", "dfs::raster_order(",
    "dfs::hilbert3d_order(", "dfs::hilbert2d_order(", "dfs::block3d_order(", "dfs::order_tokens(",
    "dfs::apply_permutation(", "dfs::invert_permutation(",
    "dfs::mean_pool(", "dfs::subblock_scores(", "dfs::aggregate_scores(", "dfs::topk_count(", "dfs::top_indices(",
    "dfs::topk_select(", "dfs::block_scores(", "dfs::build_mask(",
    "dfs::full_attention(", "dfs::full_attention_output(", "dfs::attention_scores(",
    "dfs::block_sparse_attention(", "dfs::masked_scores(", "dfs::attention_recall(",
    "dfs::SparsitySchedule::SparsitySchedule(", "dfs::SparsitySchedule::budget_at(",
    "dfs::SparsitySchedule::is_update_step(", "dfs::MaskCache::find(", "dfs::MaskCache::contains(",
    "dfs::MaskCache::store(", "dfs::MaskCache::size(", "dfs::MaskCache::clear(", "dfs::should_update(",
    "dfs::run_step(", "dfs::run_trajectory(",
]


def test_shim_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    missing = [s for s in EXPECTED if s not in out]
    assert not missing, missing


def test_headers_compile_standalone(tmp_path):
    src = tmp_path / "use.cpp"
    src.write_text("#include \"dfs/scheduler.hpp\"\n#include \"dfs/attention.hpp\"\n#include \"dfs/parallel.hpp\"\n"
                   "int main() { dfs::Matrix m(2, 3, 1.f); dfs::BlockMask b(2, 4, true);\n"
                   "  return (m.size() == 6 && b.selected_count() == 4 && dfs::block_count_for(5, 4) == 2) ? 0 : 1; }\n")
    exe = tmp_path / "use"
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    assert subprocess.run([str(exe)]).returncode == 0
