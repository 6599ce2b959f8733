"""Host-side serving contracts mirrored from the reference's own tests
(ref tests/test_pipeline.py: TestHashTableQueue, TestFidelity,
TestReportSerialization). No GPU: tables are host-built, reports are
constructed directly."""

import csv
import json
import threading

import numpy as np
import pytest

from paper_2310_18859_b200.errors import ContractError
from paper_2310_18859_b200.pipeline import HashTableQueue, ServingReport, fidelity
from paper_2310_18859_b200.predictor import ExpertHashTable


def _table(i):
    return ExpertHashTable(i, [1], np.zeros((1, 1, 1), dtype=np.int64), np.ones((1, 1, 1)))


class TestHashTableQueue:
    def test_capacity_validation(self):
        with pytest.raises(ContractError):
            HashTableQueue(0)

    def test_order_enforced_on_get(self):
        q = HashTableQueue(4)
        q.put(_table(1))
        with pytest.raises(ContractError):
            q.get(0, timeout=1.0)

    def test_order_enforced_on_put(self):
        q = HashTableQueue(4)
        q.put(_table(2))
        with pytest.raises(ContractError):
            q.put(_table(1))

    def test_fifo_round_trip(self):
        q = HashTableQueue(4)
        for i in range(3):
            q.put(_table(i))
        assert q.peek().batch_id == 0
        for i in range(3):
            assert q.get(i, timeout=1.0).batch_id == i
        assert q.peek() is None

    def test_bounded_put_blocks_until_get(self):
        q = HashTableQueue(1)
        q.put(_table(0))
        done = threading.Event()

        def producer():
            q.put(_table(1))
            done.set()

        t = threading.Thread(target=producer)
        t.start()
        assert not done.wait(0.2)  # capacity 1: the second put waits
        assert q.get(0, timeout=1.0).batch_id == 0
        assert done.wait(2.0)
        t.join()
        assert q.get(1, timeout=1.0).batch_id == 1

    def test_timeout(self):
        with pytest.raises(RuntimeError):
            HashTableQueue(2).get(0, timeout=0.05)


class TestFidelity:
    def test_identical_reports(self):
        r1 = ServingReport(mode="sida", seed=0, budget_bytes=1, eval_top_k=1, accuracy=0.8)
        r2 = ServingReport(mode="standard", seed=0, budget_bytes=1, eval_top_k=None,
                           accuracy=0.8)
        assert fidelity(r1, r2) == 1.0

    def test_zero_reference_rejected(self):
        r1 = ServingReport(mode="sida", seed=0, budget_bytes=1, eval_top_k=1, accuracy=0.5)
        r2 = ServingReport(mode="standard", seed=0, budget_bytes=1, eval_top_k=None,
                           accuracy=0.0)
        with pytest.raises(ContractError):
            fidelity(r1, r2)

    def test_unlabeled_rejected(self):
        r1 = ServingReport(mode="sida", seed=0, budget_bytes=1, eval_top_k=1)
        r2 = ServingReport(mode="standard", seed=0, budget_bytes=1, eval_top_k=None,
                           accuracy=0.5)
        with pytest.raises(ContractError):
            fidelity(r1, r2)


def test_report_json_and_csv(tmp_path):
    recs = [{"batch_id": i, "num_samples": 2, "latency_s": 0.1 * (i + 1), "queue_wait_s": 0.0,
             "transfer_s": 0.01, "compute_s": 0.05, "selection_s": 0.0} for i in range(4)]
    rep = ServingReport(mode="sida", seed=3, budget_bytes=123, eval_top_k=1, batch_records=recs,
                        throughput_samples_per_s=10.0, total_wall_s=0.8, total_samples=8,
                        hit_rate=0.75)
    rep.save_json(tmp_path / "r.json")
    rep.save_csv(tmp_path / "r.csv")
    data = json.loads((tmp_path / "r.json").read_text())
    assert data["schema_version"] == 1 and data["mode"] == "sida" and data["seed"] == 3
    assert len(data["batches"]) == 4
    assert data["aggregate"]["throughput_samples_per_s"] == 10.0
    assert data["aggregate"]["hash_hit_rate"] == 0.75
    rows = list(csv.DictReader(open(tmp_path / "r.csv")))
    assert [int(r["batch_id"]) for r in rows] == [0, 1, 2, 3]
    assert set(rows[0]) == {"batch_id", "num_samples", "latency_s", "queue_wait_s", "transfer_s",
                            "compute_s", "selection_s"}
