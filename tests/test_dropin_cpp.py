"""The C++ host layer (the reference's hisa:: entry points over the C ABI).
CPU: the library builds, links only against the C ABI and exports the reference's symbols.
GPU: paper_2603_28458_b200/cpp/test_dropin.cpp runs the SPEC examples through that API on the device."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2603_28458_b200", "_lib")


@pytest.fixture(scope="module")
def built():
    from paper_2603_28458_b200 import capi
    capi.build()
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2603_28458_b200", "cpp"), "-j4"], check=True, capture_output=True)
    return LIBDIR


def test_dropin_exports_reference_entry_points(built):
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", os.path.join(built, "libhisa_dropin.so")],
                         check=True, capture_output=True, text=True).stdout
    for sym in ["hisa::score_tokens(", "hisa::top_k_tokens(", "hisa::dsa_select(", "hisa::score_blocks(",
                "hisa::select_blocks(", "hisa::candidate_union(", "hisa::hisa_select(", "hisa::block_sparse_select(",
                "hisa::build_block_summaries(", "hisa::BlockSummaryCache::append(", "hisa::BlockSummaryCache::pooled(",
                "hisa::IndexerInputs::IndexerInputs(", "hisa::make_random_inputs(", "hisa::load_tensor_file(",
                "hisa::save_tensor_file(", "hisa::parallel_for(", "hisa::worker_count(", "hisa::analytic_cost(",
                "hisa::run_bench(", "hisa::write_bench_csv(", "hisa::to_string(", "hisa::strategy_from_string(",
                "hisa::gpu::Indexer::hisa_select_batch(", "hisa::sparse_attend(", "hisa::dense_attend(",
                "hisa::AttentionInputs::AttentionInputs(", "hisa::run_regime_equivalence_audit(",
                "hisa::run_dense_regime_audit(", "hisa::run_subset_chain_audit(", "hisa::run_overlap_ablation(",
                "hisa::gpu::Attention::sparse_attend_batch(", "hisa::generate_niah(", "hisa::selection_overlap(",
                "hisa::needle_recall(", "hisa::run_niah_grid(", "hisa::write_niah_csv(", "hisa::write_niah_grid_dat("]:
        assert sym in out, f"{sym} not exported by libhisa_dropin.so"


def test_dropin_host_layer_has_no_cuda_dependency_of_its_own(built):
    # the C++ layer reaches the device only through hisa_cuda_* (the thin C ABI)
    und = subprocess.run(["nm", "-D", "--undefined-only", os.path.join(built, "libhisa_dropin.so")],
                         check=True, capture_output=True, text=True).stdout
    assert "hisa_cuda_hisa_select" in und and "hisa_cuda_create" in und
    assert "cudaMalloc" not in und and "cuLaunch" not in und


def test_host_layer_without_a_gpu(built):
    """cpp/test_host.cpp: value types, validation rules, the RNG stream against the reference-compiled golden values,
    index arithmetic, metrics, HSB files, fan-out — everything in the C++ layer that is host code runs here on CPU."""
    r = subprocess.run([os.path.join(built, "test_host")], capture_output=True, text=True, timeout=120)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0 and "PASSED" in r.stdout, r.stdout[-3000:]


@pytest.mark.gpu
def test_dropin_spec_examples_on_gpu(built):
    r = subprocess.run([os.path.join(built, "test_dropin")], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "PASSED" in r.stdout


# ---- boundary fidelity: the C++ layer is written against the reference's OWN headers --------------------------------
REF_INC = "/root/reference/proj/core/include"
CPP_DIR = os.path.join(ROOT, "paper_2603_28458_b200", "cpp")
TUS = ["hisa_gpu.cpp", "hisa_consumer.cpp", "hisa_niah.cpp", "hisa_multi.cpp", "test_dropin.cpp", "test_host.cpp"]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_INC, "hisa")), reason="reference tree not present (GPU box)")
@pytest.mark.parametrize("tu", TUS)
def test_translation_units_compile_against_the_reference_headers(tu):
    """Every translation unit of the drop-in (and its callers' test programs) compiles with the reference's
    proj/core/include AHEAD of this repository's include/: all hisa::* declarations come from the reference, only
    hisa_gpu.hpp (namespace hisa::gpu) and hisa_cuda.h (the C ABI) come from here."""
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror", "-M", f"-I{REF_INC}",
                        f"-I{os.path.join(ROOT, 'include')}", os.path.join(CPP_DIR, tu)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    deps = r.stdout.replace("\\\n", " ").split()
    ours = [d for d in deps if os.path.abspath(d).startswith(os.path.join(ROOT, "include") + os.sep)]
    assert set(os.path.basename(d) for d in ours) <= {"hisa_cuda.h", "hisa_gpu.hpp"}, ours
    assert any(d.startswith(REF_INC) for d in deps), "no reference header was used"
    # and the same unit really compiles (not only preprocesses) in that configuration
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror", f"-I{REF_INC}",
                        f"-I{os.path.join(ROOT, 'include')}", os.path.join(CPP_DIR, tu)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]


@pytest.mark.parametrize("tu", TUS)
def test_translation_units_compile_against_the_stand_in_headers(tu):
    """Without the reference tree (the GPU box), include/hisa/*.hpp restate the same declarations."""
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                        f"-I{os.path.join(ROOT, 'include')}", os.path.join(CPP_DIR, tu)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
