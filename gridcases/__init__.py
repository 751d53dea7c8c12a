"""gridcases — benchmark case files: the seeded synthetic "-shaped" grids of
BASELINE.json's configs (``gridcases.synth``).  Plain numpy; shared by both
bench arms and the tests, so the reference arm never imports the product."""
