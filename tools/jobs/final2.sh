bash tools/jobs/final1.sh
bash tools/jobs/prof_final.sh
