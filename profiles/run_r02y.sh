# r02y: evidence set for the shared-exp loss, 10x2 fp64 gather ring and reciprocal bias corrections
bash profiles/run_evidence.sh r02y
