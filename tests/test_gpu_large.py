"""Memory scaling at the paper's SNP count (PAPER.md: 40,000 SNPs): the
narrow pair index (16 B x M^2 = 25.6 GB) fits one B200, windows of the
triple-rank space search exactly (hits re-scored by the oracle), and a
dataset whose pair index cannot fit is refused up front with E3_OOM."""
import pytest

import py_oracle as po
from paper_2201_10956_b200 import epi3


@pytest.mark.gpu
def test_40000_snps_search_windows_exact():
    M, N = 40_000, 1024
    plant = epi3.PlantSpec((7, 19_000, 38_000), (1, 1, 1), 0.9, 0.3)
    geno, pheno = epi3.generate_synthetic(M, N, 0.3, 4000, plant, exact_cases=N // 2)
    ds = epi3.binarize(geno, pheno)
    od = po.OracleDataset.of(ds)
    total = epi3.num_combinations(M, 3)
    planted = po.triple_rank(M, (7, 19_000, 38_000))
    with epi3.DeviceDataset(ds) as dd:
        for a, b in ((0, 5_000_000), (total // 2, total // 2 + 5_000_000),
                     (planted - 2_000_000, planted + 2_000_000)):
            r = dd.search(epi3.SearchConfig(top_k=10, rank_begin=a, rank_end=b))
            assert r.stats.combinations_evaluated == b - a
            for h in r.top:
                assert od.score(h.triple).hex() == h.score.hex(), h
                assert a <= po.triple_rank(M, h.triple) < b
        r = dd.search(epi3.SearchConfig(top_k=1, rank_begin=planted - 2_000_000,
                                        rank_end=planted + 2_000_000))
        assert r.best.triple == (7, 19_000, 38_000)


@pytest.mark.gpu
def test_pair_index_that_cannot_fit_is_refused_up_front():
    geno, pheno = epi3.generate_synthetic(120_000, 64, 0.3, 1, None, exact_cases=32)
    ds = epi3.binarize(geno, pheno)
    with pytest.raises(epi3.DeviceError, match="pair index"):
        epi3.DeviceDataset(ds)
