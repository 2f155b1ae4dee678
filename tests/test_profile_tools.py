"""The profile tooling behind bench.py's `traffic` fields: scripts/traffic_json.py
turns an ncu summary into profiles/ncu_traffic.json (DRAM and L2->SM bytes per
launch for each bench label), and the committed JSON agrees with the
committed summary it names."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SUMMARY = """-----
  kernel: void unnamed>::k_fbb_tma<4>(const float *, ...
  duration                 139.0 us   [gpu__time_duration.sum]
  dram read                561.019136 Mbyte   [dram__bytes_read.sum]
  dram write               7.1 Mbyte   [dram__bytes_write.sum]
  L2->L1 bytes             0.562419 Gbyte   [l1tex__m_xbar2l1tex_read_bytes.sum]
-----
  kernel: void unnamed>::k_bv_gcn1<7>(const unsigned long *, ...
  duration                 678.8 us   [gpu__time_duration.sum]
  dram read                505.735168 Mbyte   [dram__bytes_read.sum]
  dram write               29.75 Mbyte   [dram__bytes_write.sum]
  L2->L1 bytes             7.837464 Gbyte   [l1tex__m_xbar2l1tex_read_bytes.sum]
"""


def test_traffic_json_parses_a_summary(tmp_path):
    src = tmp_path / "summary.txt"
    src.write_text(SUMMARY)
    (tmp_path / "profiles").mkdir()
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "traffic_json.py"), str(src)], check=True,
                   cwd=tmp_path, capture_output=True)
    d = json.loads((tmp_path / "profiles" / "ncu_traffic.json").read_text())
    assert d["layer0.mm[BMM.FBB]"]["traffic_bytes"] == 561_019_136 + 7_100_000
    assert d["layer1.spmm[BSpMM.FBF]"]["l2_to_l1_bytes"] == 7_837_464_000
    assert "k_bv_gcn1" in d["layer1.spmm[BSpMM.FBF]"]["kernel"]


def test_committed_traffic_json_matches_its_summary():
    d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    for label, rec in d.items():
        src = rec["source"].split(" ")[0]
        assert os.path.exists(os.path.join(ROOT, src)), src
        assert rec["traffic_bytes"] == rec.get("dram_read", 0) + rec.get("dram_write", 0)
