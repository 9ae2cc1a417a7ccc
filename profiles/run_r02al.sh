# r02al: final evidence set of the round (GPU suite, smoke, bench, reference arm, 2-rank gloo, full-workload ncu)
bash profiles/run_evidence.sh r02al
