python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python scripts/exp/workers_probe.py
python scripts/exp/dropin_probe.py | tail -3
cd baseline/_ref_tests && PYTHONPATH=../_ref:../.. python -m pytest -q -p paper_1506_08503_b200.plugin -p no:cacheprovider --rootdir . test_acceptance.py -k criterion_8 2>&1 | grep -E "criterion 8|passed|failed"
