for w in 1 2 4; do for srt in none deg; do echo "W=$w sort=$srt"; python tools/prof_batch.py --sources 1024 --lane-words $w --sort $srt --repeat 2 | tail -1; done; done
