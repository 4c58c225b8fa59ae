"""Host logic of the optimizer orchestration (paper_2206_15397_b200/kfac.py) against the reference's rules
(optimizer.hpp:38-121, network.hpp:82-91)."""
import pytest

from paper_2206_15397_b200.kfac import (ConfigError, Method, OptimizerConfig, ScheduleOverrides, factor_statistics,
                                        needs_recompute, run_schedules)


@pytest.mark.parametrize("epoch,t_ki,lam,alpha,r,p", [
    (0, 50, 0.1, 0.3, 220, 10),
    (2, 50, 0.1, 0.2, 220, 10),
    (3, 50, 0.1, 0.1, 220, 10),
    (15, 50, 0.1, 0.03, 230, 10),
    (20, 30, 0.1, 0.01, 230, 10),
    (22, 30, 0.1, 0.01, 230, 11),
    (25, 30, 0.05, 0.01, 230, 11),
    (30, 30, 0.05, 0.003, 230, 12),
    (35, 30, 0.01, 0.003, 230, 12),
    (40, 30, 0.01, 0.001, 230, 12),
])
def test_schedules_follow_optimizer_hpp(epoch, t_ki, lam, alpha, r, p):
    s = run_schedules(OptimizerConfig(), epoch)
    assert (s.t_ki, s.target_rank, s.oversampling) == (t_ki, r, p)
    assert s.lam == pytest.approx(lam, abs=1e-12) and s.alpha == pytest.approx(alpha, abs=1e-12)


def test_schedule_overrides_and_errors():
    cfg = OptimizerConfig(overrides=ScheduleOverrides(lam=0.5, target_rank=64, oversampling=4, t_ki=20, alpha=1.0))
    s = run_schedules(cfg, 40)
    assert (s.lam, s.target_rank, s.oversampling, s.t_ki, s.alpha) == (0.5, 64, 4, 20, 1.0)
    with pytest.raises(ConfigError):
        run_schedules(OptimizerConfig(t_ku=60), 0)  # T_KI < T_KU
    with pytest.raises(ConfigError):
        run_schedules(OptimizerConfig(overrides=ScheduleOverrides(lam=0.0)), 0)
    with pytest.raises(ConfigError):
        OptimizerConfig(rho=1.0).validate()
    with pytest.raises(ConfigError):
        OptimizerConfig(t_ku=0).validate()


def test_needs_recompute():
    assert needs_recompute(None, 7, 50, "srevd")
    assert needs_recompute("rsvd", 7, 50, "srevd")
    assert needs_recompute("srevd", 100, 50, "srevd")
    assert not needs_recompute("srevd", 101, 50, "srevd")


def test_factor_statistics_appends_the_ones_row():
    import torch

    a = torch.randn(5, 8)
    d = torch.randn(3, 8)
    am, gm = factor_statistics([a], [d])
    assert am[0].shape == (6, 8) and torch.equal(am[0][:5], a) and torch.equal(am[0][5], torch.ones(8))
    assert gm[0] is d
    assert Method.SRE_KFAC.value == 2


def test_runlog_and_spectrum_csv_schema(tmp_path):
    from paper_2206_15397_b200.kfac import (SpectrumReport, SpectrumSnapshot, StepRecord, StepTimings, decay_orders,
                                            write_runlog_csv, write_spectrum_csv)

    write_runlog_csv(str(tmp_path / "runlog.csv"), [StepRecord(0, 0, 2.5, -1.0, StepTimings(0.1, 0.2, 0.3))])
    assert (tmp_path / "runlog.csv").read_text().splitlines() == [
        "step,epoch,loss,acc,t_factor,t_decomp,t_apply", "0,0,2.5,-1,0.10000000000000001,0.20000000000000001,"
        "0.29999999999999999"]
    write_spectrum_csv(str(tmp_path / "spectrum.csv"), [SpectrumSnapshot(3, 1, [2.0, 0.5])])
    assert (tmp_path / "spectrum.csv").read_text().splitlines() == ["step,layer,idx,eigenvalue", "3,1,0,2", "3,1,1,0.5"]
    assert decay_orders([100.0, 10.0, 1.0], 3) == pytest.approx(2.0)
    assert decay_orders([1.0, 0.0], 2) == 300.0 and decay_orders([], 5) == 0.0
    rep = SpectrumReport([4.0, 2.0, 0.5, 0.0], 4.0)
    assert rep.count_above(0.1) == 3


def test_conv_output_size_matches_the_convolution_arithmetic():
    from paper_2206_15397_b200.kfac import conv_output_size

    assert conv_output_size(32, 32, 3, 1, 1) == (32, 32)  # VGG16 3x3, padding 1
    assert conv_output_size(8, 8, 3, 2, 1) == (4, 4)
    assert conv_output_size(7, 9, (3, 1), (2, 1), (0, 0), (2, 1)) == (2, 9)
