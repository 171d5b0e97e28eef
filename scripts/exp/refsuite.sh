cd baseline/_ref_tests
PYTHONPATH=../_ref:../.. python -m pytest -q -p paper_1506_08503_b200.plugin -p no:cacheprovider --rootdir . test_cli.py test_bench.py 2>&1 | tail -15
PYTHONPATH=../_ref:../.. python -m pytest -q -p paper_1506_08503_b200.plugin -p no:cacheprovider --rootdir . test_acceptance.py -k criterion_8 2>&1 | tail -15
