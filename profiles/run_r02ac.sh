# r02ac: evidence set with the concurrent single-contribution rows (12-item tiles)
bash profiles/run_evidence.sh r02ac
